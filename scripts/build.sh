#!/bin/sh
# rebuild libch_b200.so in-tree (same as __graft_entry__.build())
cd "$(dirname "$0")/.." && python -c "
import importlib.util
spec = importlib.util.spec_from_file_location('b', 'paper_1811_11842_b200/build.py')
m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" && echo built
