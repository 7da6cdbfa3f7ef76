"""bench.py contract (CPU): the metric's numerator and byte model against SURVEY §8(d)'s
table (algorithmic F+SI TFLOP and GB per config), and the reference arm's JSON line on
the tiny config C1 (the reference arm is the CPU oracle; no GPU needed)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

# Flops F + SI (TFLOP), Bytes F + SI (GB)
TABLE = {"C2": (0.345, 0.689, 8.8), "C3": (7.32, 14.63, 98), "C5": (0.0117, 0.0234, 4.56)}


@pytest.mark.parametrize("cfg", sorted(TABLE))
def test_algorithmic_work_matches_survey_table(cfg):
    n, b, a = (bench.CONFIGS[cfg][k] for k in ("n", "b", "a"))
    F, S, B = TABLE[cfg]
    assert bench.flops_pobtaf(n, b, a) / 1e12 == pytest.approx(F, rel=0.01)
    assert bench.flops_pobtasi(n, b, a) / 1e12 == pytest.approx(S, rel=0.01)
    assert bench.algorithmic_bytes(n, b, a) / 1e9 == pytest.approx(B, rel=0.01)


def test_flops_per_block_leading_order():
    # (n-1)(7/3 + 14/3) b^3 = 7 b^3 per block for a = 0 at large n (LAPACK counting)
    n, b = 1000, 64
    per = (bench.flops_pobtaf(n, b, 0) + bench.flops_pobtasi(n, b, 0)) / (n * b ** 3)
    assert per == pytest.approx(7.0, rel=2e-3)


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "TFLOP/s" and line["value"] > 0
    assert line["higher_is_better"] is True and line["dtype"] == "f64"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["config"]["workload"].startswith("C1")
