"""bench.py's host-side pieces: the BASELINE workloads' scenes and initial
states (configs[1], [3], [4]) and the JSON contract of the reference arm."""

import json
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2009_14514_b200.scene import seed_particles  # noqa: E402


def test_cfg2_scene_counts():
    f, w = seed_particles(bench.scene_cfg2())
    assert len(f) == 1_000_000 and len(w) == 510_064


def test_cfg4_mixed_tank_geometry():
    sc = bench.scene_cfg4()
    assert sc.gravity == (0.0, 0.0, -9.81)
    f, _ = seed_particles(sc)
    v = bench.initial_velocity("cfg4", f)
    block = v[:, 2] < 0
    assert len(f) == 8_015_190
    # 80 / 20 split, block 1 m above the pool, below the lid
    assert abs(block.mean() - 0.2) < 0.005
    assert f[~block, 2].max() < 2.0 / 3.0
    assert abs(f[block, 2].min() - f[~block, 2].max() - 1.0) < 2 * sc.spacing
    assert f[block, 2].max() < 2.0
    assert np.all(v[block] == (0.0, 0.0, -2.0)) and np.all(v[~block] == 0.0)


def test_cfg5_weak_scaling_scene():
    for world in (1, 2):
        for kind in ("pcisph", "wcsph"):
            sc = bench.scene_cfg5(world, kind)
            f, _ = seed_particles(sc)
            assert len(f) == 4_000_000 * world
    f, _ = seed_particles(bench.scene_cfg5(1))
    v = bench.initial_velocity("cfg5-pcisph", f)
    assert abs(float(v.std()) - 0.1) < 1e-3 and abs(float(v.mean())) < 1e-3
    # seeded: identical on every call (every rank draws the same field)
    assert np.array_equal(v, bench.initial_velocity("cfg5-wcsph", f))


def test_reference_arm_other_ranks_exit_quietly():
    import os
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_workload_table_is_complete():
    for name, (kind, desc, scaling) in bench.WORKLOADS.items():
        assert kind in ("pcisph", "wcsph") and scaling in ("weak", "strong")
        assert name in bench.METRICS and desc.startswith(name.split("-")[0])
    json.dumps(bench.WORKLOADS)


def test_reference_arm_bounded_sample():
    """--impl reference: one JSON line on the same config; past the wall
    budget it reports the steps it actually timed (a bounded sample)."""
    import os
    env = dict(os.environ, RTS_REF_BUDGET_S="0.001")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "3", "--warmup", "0"],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["steps"] == 1 and d["steps_requested"] == 3
    assert "bounded sample" in d["cpu_baseline"]["sample"] and d["value"] > 0
    assert d["config"] == bench.bench_config("cfg2", 1, d["config"]["n_fluid"],
                                             d["config"]["n_boundary"])
    assert d["e2e"]["value"] == d["value"]
