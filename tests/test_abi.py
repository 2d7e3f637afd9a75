"""The C-ABI library loads and exports every symbol include/gasb.h declares (CPU)."""
import re
from pathlib import Path

import paper_2106_05609_b200 as gb

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "gasb.h").read_text()
    return sorted(set(re.findall(r"\b(gasb_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    syms = declared_symbols()
    assert len(syms) > 40
    missing = [s for s in syms if not hasattr(gb.lib, s)]
    assert not missing, missing


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(gb.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_error_status_maps_to_reference_exception():
    import pytest
    with pytest.raises(ValueError):
        gb.build_graph([[0, 9]], 2)
    assert "out of range" in gb.lib.gasb_last_error().decode()


def _build_shim_test(tmp_path):
    import subprocess
    exe = tmp_path / "test_shim"
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Werror", f"-I{ROOT / 'include'}", str(ROOT / "tests" / "cpp" / "test_shim.cpp"),
           "-o", str(exe), f"-L{gb.LIB_PATH.parent}", "-lgasb", f"-Wl,-rpath,{gb.LIB_PATH.parent}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_shim_host_parts(tmp_path):
    """include/gasb/gas.hpp compiles -Werror against gasb.h, links libgasb.so, and its host parts
    (Graph, BatchSchedule, error mapping) pass; device parts fail loudly without a GPU."""
    import subprocess
    r = subprocess.run([str(_build_shim_test(tmp_path))], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
