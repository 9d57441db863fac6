"""GPU: run_simulation with the B200 solvers (reference pkg/tests/test_bench.py)."""

import json

import numpy as np
import pytest

from conftest import tiny_tank

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["wcsph", "wcsph-rts", "pcisph-const", "pcisph-adaptive",
                                  "pcisph-rts"])
def test_run_directory_layout(tmp_path, name):
    from paper_2009_14514_b200.run import frame_files, read_frame, run_simulation
    meta = run_simulation(tiny_tank(), name, duration=0.01, fps=200, out_dir=tmp_path)
    files = frame_files(tmp_path)
    assert len(files) == meta["n_frames"] == 2
    t0, pos0, reg0 = read_frame(files[0])
    assert t0 == 0.0 and pos0.shape == (meta["n_fluid"], 3)
    assert (tmp_path / "stats.csv").exists()
    assert json.loads((tmp_path / "meta.json").read_text())["solver"] == name
    assert meta["steps"] > 0 and meta["wall_time"] > 0


def test_identical_runs_write_identical_frames(tmp_path):
    from paper_2009_14514_b200.run import compare, frame_files, run_simulation
    a, b = tmp_path / "a", tmp_path / "b"
    run_simulation(tiny_tank(), "pcisph-rts", duration=0.02, fps=100, out_dir=a)
    run_simulation(tiny_tank(), "pcisph-rts", duration=0.02, fps=100, out_dir=b)
    for fa, fb in zip(frame_files(a), frame_files(b)):
        assert fa.read_bytes() == fb.read_bytes()
    r = compare(a, b)
    assert r["com_deviation"] == 0.0 and r["work_ratio"] == 1.0


def test_frames_hold_the_state_of_their_step_at_scale(tmp_path):
    """a frame copies the state of the step it belongs to even
    when the copy outlasts a step (1 M particles, a frame after every major
    step): the exporter snapshots pos / region on the compute stream before
    its side-stream copy, so the next advance() cannot overwrite them.
    Compared with a second, deterministic run read synchronously."""
    import bench
    from paper_2009_14514_b200 import PcisphSolver
    from paper_2009_14514_b200.run import frame_files, read_frame, run_simulation
    sc = bench.scene_cfg2()
    dt = sc.base_dt("pcisph")
    major = 4 * dt
    run_simulation(sc, "pcisph-rts", duration=3 * major, fps=int(round(1.0 / major)),
                   out_dir=tmp_path, frames_only=True, solver_kwargs={"iteration_cap": 50})
    ref = PcisphSolver(sc, mode="rts", iteration_cap=50)
    frames = [read_frame(f) for f in frame_files(tmp_path)]
    assert len(frames) >= 3
    t0, p0, _ = frames[0]
    assert t0 == 0.0 and np.array_equal(p0, ref.host("pos")[: ref.n_fluid].astype(np.float32))
    for t, pos, reg in frames[1:]:
        while ref.sim_time < t - 1e-12:
            ref.advance()
        assert ref.sim_time == pytest.approx(t, rel=1e-12)
        assert np.array_equal(pos, ref.host("pos")[: ref.n_fluid].astype(np.float32))
        assert np.array_equal(reg, ref.particle_regions().cpu().numpy().astype(np.uint8))
