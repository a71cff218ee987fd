mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> $S
timeout 900 python bench.py > gpurun_out/bench_final4.log 2>&1; echo bench=$? >> $S
