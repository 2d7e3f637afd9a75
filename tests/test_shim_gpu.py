"""The C++ shim's device parts (HistoryStore push/pull/stamps/errors) on a GPU."""
import subprocess

import pytest

from test_abi import _build_shim_test

pytestmark = pytest.mark.gpu


def test_cpp_shim_device_parts(tmp_path):
    r = subprocess.run([str(_build_shim_test(tmp_path))], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("gpu 0 failures"), r.stdout
