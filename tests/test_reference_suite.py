"""The reference's own test suites, re-run through the drop-in.

`binfec.{field, basis, transform, derivative, walsh, rs, batch}` are
redirected to this repo's GPU shim (tests/refsuite/binfec_shim_plugin.py)
before the reference's conftest imports them, and the unmodified test files
run: results, exception types, return types, OpCounter totals and
ErasurePattern semantics are checked by the reference's own assertions.

The suite and the reference package are staged into the git-ignored
baseline/_ref/ by tools/stage_reference.sh (this container); the test skips
when they are absent.
"""

import os
import re
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "ref_tests")

SUITES = ["test_transform.py", "test_rs.py", "test_batch.py", "test_walsh.py",
          "test_derivative.py", "test_field.py", "test_basis.py"]


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_through_shim(suite, tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.isfile(os.path.join(REF_TESTS, suite)):
        pytest.skip("reference suite not staged (tools/stage_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(HERE, "refsuite"), REF_TESTS, ROOT,
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-p", "binfec_shim_plugin", "-q", "-p", "no:cacheprovider",
           "--rootdir", REF_TESTS, "-o", "addopts=", os.path.join(REF_TESTS, suite)]
    res = subprocess.run(cmd, cwd=str(tmp_path), env=env, capture_output=True, text=True, timeout=1500)
    tail = "\n".join(res.stdout.splitlines()[-25:])
    print(tail)
    assert res.returncode == 0, f"{suite} through the shim:\n{tail}\n{res.stderr[-2000:]}"
    m = re.search(r"(\d+) passed", res.stdout)
    assert m and int(m.group(1)) > 0
