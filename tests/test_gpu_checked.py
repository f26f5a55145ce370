"""GPU: every kernel path under the bounds-checked build (`make checks`,
-DPSG_CHECKS). compute-sanitizer is not available on this GPU pool, so the ring
allocation, record-block, list-position, bin-scatter and plane-index invariants
are asserted on the device instead; a failed check traps and the run fails.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2412_03451_b200", "lib", "libpsplat_b200_checks.so")


@pytest.mark.gpu
def test_all_kernel_paths_under_bounds_checks():
    if not os.path.exists(CHECKED):
        pytest.skip("checked build absent (make -C paper_2412_03451_b200/csrc checks)")
    product = os.path.join(ROOT, "paper_2412_03451_b200", "lib", "libpsplat_b200.so")
    if os.path.exists(product) and os.path.getmtime(CHECKED) < os.path.getmtime(product):
        pytest.fail("the checked build is older than the product library: "
                    "run make -C paper_2412_03451_b200/csrc checks (build() does)")
    env = dict(os.environ, PSG_LIB=CHECKED)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_case.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "sanitize_case: ok True" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
    # the full-size C3 step at the lowest lambda of the schedule (crowded tiles,
    # full per-pixel lists) and at lambda 300
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "profile_step.py"), "--views", "32",
                        "--lam", "7.36,300", "--precision", "fp64", "--reps", "1"], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.count("views/s raster-only") == 2, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_cull_audit_no_misses():
    """Checked build: every candidate rejected by the footprint rect or the fp32 cull
    is re-tested with the exact fp64 test on stratified C3 views (every 32nd) and
    C5 views (every 64th) across the schedule's lambda range; no miss and no
    depth-bound violation is allowed. The whole-workload run (1024 C3 and 256 C5
    views) is committed in profiles/ (scripts/cull_audit.py)."""
    import json
    if not os.path.exists(CHECKED):
        pytest.skip("checked build absent (make -C paper_2412_03451_b200/csrc checks)")
    env = dict(os.environ, PSG_LIB=CHECKED)
    for cfg, stride in (("c3", 32), ("c5", 64)):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "cull_audit.py"), "--config", cfg,
                            "--stride", str(stride), "--lams", "7.3576,20,300"], env=env,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        res = json.loads(r.stdout.strip().splitlines()[-1])
        print("\n" + json.dumps(res))
        assert res["ok"], res

