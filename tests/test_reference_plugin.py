"""The reference's own test files against the B200 path:
integration/plugin.py patches the unmodified reference installed in
baseline/_ref (tools/install_reference.sh) so that
  * mode "kernel": every pac() of the reference goes through codec_pac on
    the GPU (its compiled-kernel boundary, _kernels.pyx:16-18);
  * mode "execute": execute() runs the whole decode step on the GPU.
The reference's test_kernels / test_attention / test_executor /
test_acceptance must pass, and the plugin must have been called."""
from __future__ import annotations

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
REF_TESTS = ROOT / "baseline" / "_ref" / "tests"
FILES = ["test_kernels.py", "test_attention.py", "test_executor.py", "test_acceptance.py"]


@pytest.mark.parametrize("mode", ["kernel", "execute"])
def test_reference_suite_on_b200(cuda_ok, mode):
    if not REF_TESTS.exists():
        pytest.skip("baseline/_ref not installed (tools/install_reference.sh)")
    env = dict(os.environ, B200_PLUGIN_MODE=mode)
    res = subprocess.run([sys.executable, "-m", "pytest", "-p", "integration.plugin", "-p", "no:cacheprovider", "-q",
                          *[str(REF_TESTS / f) for f in FILES]], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=900)
    tail = res.stdout[-3000:]
    assert res.returncode == 0, tail
    calls = re.search(r"B200 plugin calls: \{'pac_kernel': (\d+), 'execute': (\d+)\}", res.stdout)
    assert calls, tail
    assert int(calls.group(1)) > 1000
    if mode == "execute":
        assert int(calls.group(2)) > 100
