"""CPU: bench.py's contract pieces that need no GPU -- the algorithmic bytes of
SURVEY.md 8d, the structure-overhead and compute-fraction models, and the
reference arm's JSON line (`bench.py --impl reference`, oracle/_ref on the host)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_algorithmic_bytes_match_survey():
    # B_v = 36 W H + 44 P -> 11.15 / 11.50 / 47.36 MB
    assert bench.algorithmic_bytes_per_view(640, 480, 2000) == 11_147_200
    assert bench.algorithmic_bytes_per_view(640, 480, 10000) == 11_499_200
    assert bench.algorithmic_bytes_per_view(1296, 968, 50000) == 47_363_008


def test_structure_overhead_model():
    o = bench.structure_overhead_per_view(640, 480, 244246.0)
    px = 640 * 480
    assert o["maps_reread"] == 20 * px and o["dmaps_write_read"] == 32 * px
    assert o["record_lists_write_read"] == 2 * (2 * px + 4 * 244246.0)
    assert o["bytes_per_view"] == o["maps_reread"] + o["dmaps_write_read"] + o["record_lists_write_read"]
    assert o["in_roofline"] is False


def test_compute_fraction_model():
    st = {"views": 2, "pixel_pairs": 2 * 1000, "live_records": 2 * 10}
    c = bench.compute_fraction(st, 1.0, 1965.0)
    assert c["Q_v"] == 1000 and c["L_v"] == 10
    assert c["F_v_fp32_ops"] == 28 * 1000 + 250 * 10 and c["X_v_mufu_ops"] == 1000 + 4 * 10
    fp32 = 148 * 128 * 2 * 1965e6
    mufu = 148 * 16 * 1965e6
    want = max(c["F_v_fp32_ops"] / fp32, c["X_v_mufu_ops"] / mufu) / 1e-3
    assert abs(c["frac_at_1965MHz"] - want) <= 1e-12 * want


def test_reference_arm_json_line():
    from oracle.oracle import LIBS
    if not os.path.exists(LIBS["ref"]):
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "views/s"
    assert line["steps"] == 2 and line["warmup"] == 1 and line["higher_is_better"] is True
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["value"] == line["value"] and cb["cores"] >= 1 and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "views/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["metric"] == "views/sec fwd+bwd planar splat"


def test_gpus_flag_never_downgrades(tmp_path):
    """bench.py --gpus N launches N ranks itself when no torchrun environment is set,
    refuses (exit 2) when fewer than N GPUs are visible, and refuses a WORLD_SIZE that
    differs from --gpus (no silent one-rank run)."""
    import subprocess
    import sys
    bench = os.path.join(ROOT, "bench.py")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, bench, "--gpus", "2", "--steps", "1", "--warmup", "1"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "only 0 CUDA device" in r.stderr, r.stderr[-500:]
    env2 = dict(env, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, bench, "--gpus", "4"], env=env2, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr, r.stderr[-500:]
