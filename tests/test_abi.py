"""The C-ABI library loads and exports every symbol include/ch_b200.h declares;
the ctypes structs match the C layout (-m "not gpu": no compute calls)."""
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "ch_b200.h")


def _declared():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ch_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_1811_11842_b200 import _lib
    names = _declared()
    assert len(names) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (ch_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(_lib.EXPORTS) == set(names)
    assert _lib.lib.ch_abi_version() == 2


def test_ctypes_struct_layout_matches_c(tmp_path):
    from paper_1811_11842_b200 import _lib
    import ctypes
    src = tmp_path / "sz.c"
    src.write_text('#include "ch_b200.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(ch_grid), '
                   'sizeof(ch_params), sizeof(ch_stats), offsetof(ch_params, maxit), '
                   'offsetof(ch_stats, kc_ms), offsetof(ch_params, theta_visc), '
                   'offsetof(ch_params, startup_be));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert vals == [ctypes.sizeof(_lib.Grid), ctypes.sizeof(_lib.Params), ctypes.sizeof(_lib.Stats),
                    _lib.Params.maxit.offset, _lib.Stats.kc_ms.offset,
                    _lib.Params.theta_visc.offset, _lib.Params.startup_be.offset]


def test_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1811_11842_b200 import Simulation, CHError
    with pytest.raises(CHError):
        Simulation(16, 16)


def test_bad_arguments_rejected_before_device_work():
    from paper_1811_11842_b200 import Simulation, CHError
    with pytest.raises(CHError):
        Simulation(2, 16)           # nx < 4
    with pytest.raises(CHError):
        Simulation(17, 16)          # odd nx (two columns per thread)
    with pytest.raises(CHError):
        Simulation(16, 16, theta_visc=0.0)
    with pytest.raises(CHError):
        Simulation(16, 16, dt=-1.0)


def test_field_ids_match_header(tmp_path):
    from paper_1811_11842_b200 import _lib
    names = ["PHI", "PHI_PREV", "C", "U", "V", "P", "U_STAR", "V_STAR"]
    src = tmp_path / "f.c"
    src.write_text('#include "ch_b200.h"\n#include <stdio.h>\nint main(void){'
                   + "".join(f'printf("%d\\n", CH_FIELD_{n});' for n in names) + "return 0;}\n")
    exe = tmp_path / "f"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert vals == [_lib.FIELDS[n.lower()] for n in names]
