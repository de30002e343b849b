"""Checked mode (WFK_CHECK=1, include/wfk.h): libwfk's own memcheck /
initcheck stand-ins, since compute-sanitizer is not offered on the GPU pool.
Every device buffer is poisoned with 0xff bytes when allocated and carries a
canary tail that every C-ABI call verifies before returning.  These tests run
in subprocesses because the mode is read once, when the library loads.

* the detector itself: a kernel writing past the end of a scratch buffer
  fails the call (and a write that stays inside does not);
* a solve / fusion / process_frame workload (tools/sanitize_fixture.py) at
  reference parity with every allocation poisoned and every canary intact.

The whole `-m gpu` suite run under WFK_CHECK=1 is the full-coverage version
(profiles/r02_checked_gpu_tests.log)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu

DETECTOR = r"""
import sys
sys.path.insert(0, sys.argv[1])
from paper_1603_08161_b200.wfk import Context, WfkError, check_enabled
assert check_enabled()
ctx = Context(0)
ctx.debug_overrun(0)           # inside the buffer: no error
for past in (1, 8, 256):
    try:
        ctx.debug_overrun(past)
    except WfkError as e:
        assert "WFK_CHECK: write past the end" in str(e), str(e)
    else:
        raise SystemExit(f"overrun of {past} bytes not detected")
ctx.debug_overrun(0)           # a fresh buffer: the context is usable again
ctx.close()
print("detector OK")
"""


def _run(args, check_env="1", timeout=600, **extra):
    env = dict(os.environ)
    env["WFK_CHECK"] = check_env
    env.update(extra)
    return subprocess.run(args, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def test_checked_mode_detects_overrun():
    out = _run([sys.executable, "-c", DETECTOR, ROOT])
    assert out.returncode == 0, out.stdout + out.stderr
    assert "detector OK" in out.stdout


def test_checked_mode_off_by_default():
    out = _run([sys.executable, "-c",
                "import sys; sys.path.insert(0, sys.argv[1]);"
                "from paper_1603_08161_b200.wfk import check_enabled; print(check_enabled())", ROOT],
               check_env="0")
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip() == "False"


@pytest.mark.parametrize("pcg", ["pipe", "cg"])
def test_checked_workload_parity(pcg):
    out = _run([sys.executable, os.path.join(ROOT, "tools", "sanitize_fixture.py")], WFK_PCG=pcg)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "sanitize fixture OK" in out.stdout
