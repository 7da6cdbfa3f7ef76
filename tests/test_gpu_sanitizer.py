"""compute-sanitizer on the library's kernels (hand-rolled acquire/release counters,
cp.async pipelines, named barriers in exec.cu; the small-block engine's in-smem
chains in sb.cu): memcheck and racecheck must report no errors on small problems of
every path -- sequential selinv (C1 shape), the partitioned graph, and the
small-block engine with nesting.
"""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np, torch
import btagen, paper_2503_17528_b200 as sb
from tests.gpu_util import to_dev, args
which = sys.argv[1]
if which == "selinv":
    D = to_dev(btagen.g1(1, 8, 4, 2)); sb.selinv(*args(D))
    D = to_dev(btagen.g1(1, 5, 70, 5)); sb.selinv(*args(D))
elif which == "pselinv":
    D = to_dev(btagen.g2(1, 24, 64, 4)); sb.pselinv(*args(D), 3)
elif which == "sb":
    D = to_dev(btagen.g2(1, 40, 64, 8)); sb.selinv_sb(*args(D), [5, 3])
    D = to_dev(btagen.g1(1, 9, 13, 3)); sb.selinv_sb(*args(D), [3])
torch.cuda.synchronize()
print("done")
"""


def _sanitizer():
    if os.environ.get("SERINV_SANITIZER") != "1":
        pytest.skip("opt-in (SERINV_SANITIZER=1): the GPU pool blocks compute-sanitizer runs "
                    "(profiles/r02/sanitizer.txt holds the last clean run)")
    for c in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if c and os.path.exists(c):
            return c
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
@pytest.mark.parametrize("which", ["selinv", "pselinv", "sb"])
def test_sanitizer_clean(tool, which):
    cs = _sanitizer()
    code = SCRIPT.format(root=ROOT)
    cmd = [cs, "--tool", tool, "--error-exitcode", "3", sys.executable, "-c", code, which]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "done" in out
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-2000:]
