"""``rts-sph-bench`` command line (paper_2009_14514_b200.cli) through main(),
mirroring the reference's tests/test_cli.py: configuration errors exit 1
before any device work (CPU), runs / compare / numerical aborts on the GPU."""

import pytest

from conftest import TINY_TANK_TEXT


@pytest.fixture
def scene_file(tmp_path):
    path = tmp_path / "tank.txt"
    path.write_text(TINY_TANK_TEXT)
    return str(path)


def run_cli(*argv):
    from paper_2009_14514_b200.cli import main
    return main(list(argv))


# ---- CPU: parsing and configuration errors --------------------------------

def test_bad_thread_env_is_a_config_error(scene_file, tmp_path, monkeypatch, capsys):
    monkeypatch.setenv("RTS_SPH_THREADS", "many")
    code = run_cli("run", "--scene", scene_file, "--solver", "wcsph",
                   "--duration", "0", "--out", str(tmp_path / "run"))
    assert code == 1
    assert "RTS_SPH_THREADS" in capsys.readouterr().err


def test_bad_thread_count_is_a_config_error(scene_file, tmp_path, capsys):
    code = run_cli("run", "--scene", scene_file, "--solver", "wcsph",
                   "--duration", "0", "--out", str(tmp_path / "run"), "--threads", "0")
    assert code == 1
    assert "thread count" in capsys.readouterr().err


def test_missing_scene_exits_one(tmp_path, capsys):
    code = run_cli("run", "--scene", str(tmp_path / "nope.txt"), "--solver", "wcsph",
                   "--duration", "0", "--out", str(tmp_path / "run"))
    assert code == 1
    assert "cannot read scene" in capsys.readouterr().err


def test_unknown_solver_exits_one(scene_file, tmp_path):
    with pytest.raises(SystemExit) as exc:
        run_cli("run", "--scene", scene_file, "--solver", "sph9000",
                "--out", str(tmp_path / "run"))
    assert exc.value.code == 1


def test_bad_minor_steps_exits_one(scene_file, tmp_path):
    with pytest.raises(SystemExit) as exc:
        run_cli("run", "--scene", scene_file, "--solver", "pcisph-rts",
                "--out", str(tmp_path / "run"), "--minor-steps", "3")
    assert exc.value.code == 1


def test_compare_rejects_non_run_directory(tmp_path, capsys):
    code = run_cli("compare", str(tmp_path), str(tmp_path))
    assert code == 1
    assert "no meta.json" in capsys.readouterr().err


def test_module_entry_point_prints_usage():
    import subprocess
    import sys
    out = subprocess.run([sys.executable, "-m", "paper_2009_14514_b200", "--help"],
                         capture_output=True, text=True, timeout=120)
    assert out.returncode == 0
    assert "rts-sph-bench" in out.stdout and "compare" in out.stdout


# ---- GPU: runs through the B200 solvers ----------------------------------

@pytest.mark.gpu
def test_run_exports_frames_and_summary(scene_file, tmp_path, capsys):
    from paper_2009_14514_b200.run import frame_files
    out = tmp_path / "run"
    code = run_cli("run", "--scene", scene_file, "--solver", "wcsph",
                   "--duration", "0.01", "--fps", "300", "--out", str(out))
    assert code == 0
    assert len(frame_files(out)) == 3
    assert (out / "stats.csv").exists()
    stdout = capsys.readouterr().out
    assert "solver wcsph on 1000 fluid particles" in stdout
    assert "3 frames" in stdout
    assert "breakdown:" in stdout


@pytest.mark.gpu
def test_zero_duration_frames_only(scene_file, tmp_path):
    from paper_2009_14514_b200.run import frame_files
    out = tmp_path / "run"
    code = run_cli("run", "--scene", scene_file, "--solver", "pcisph-rts",
                   "--duration", "0", "--out", str(out), "--frames-only")
    assert code == 0
    assert [f.name for f in frame_files(out)] == ["frame_00000.bin"]
    assert not (out / "stats.csv").exists()


@pytest.mark.gpu
def test_preset_scene_by_name(tmp_path, capsys):
    code = run_cli("run", "--scene", "dam_break", "--solver", "wcsph",
                   "--duration", "0", "--out", str(tmp_path / "run"))
    assert code == 0
    assert "8000 fluid particles" in capsys.readouterr().out


@pytest.mark.gpu
def test_minor_steps_and_audit_flags(scene_file, tmp_path, capsys):
    code = run_cli("run", "--scene", scene_file, "--solver", "pcisph-rts",
                   "--duration", "0.003", "--fps", "30", "--out", str(tmp_path / "run"),
                   "--minor-steps", "2", "--audit-neighbors", "--deterministic")
    assert code == 0
    assert "missed neighbors: 0" in capsys.readouterr().out


@pytest.mark.gpu
def test_numerical_abort_exits_two(scene_file, tmp_path, capsys):
    code = run_cli("run", "--scene", scene_file, "--solver", "wcsph-rts",
                   "--duration", "1.0", "--out", str(tmp_path / "run"), "--dt-base", "0.05")
    assert code == 2
    assert "numerical abort" in capsys.readouterr().err


@pytest.mark.gpu
def test_compare_command(scene_file, tmp_path, capsys):
    for name in ("a", "b"):
        assert run_cli("run", "--scene", scene_file, "--solver", "pcisph-const",
                       "--duration", "0.002", "--fps", "1000", "--out",
                       str(tmp_path / name)) == 0
    capsys.readouterr()
    code = run_cli("compare", str(tmp_path / "a"), str(tmp_path / "b"))
    assert code == 0
    stdout = capsys.readouterr().out
    assert "wall-clock speedup:" in stdout
    assert "work ratio:" in stdout
    assert "max COM deviation:" in stdout
    # identical deterministic runs: zero deviation
    assert "max COM deviation:   0.000000 m" in stdout


def test_reports_match_the_reference_lines():
    """run / compare summaries without a device (reference cli.py:108-138)."""
    from paper_2009_14514_b200.cli import compare_report, run_report
    meta = {"solver": "pcisph-rts", "n_fluid": 1000, "duration": 0.5, "steps": 10,
            "n_frames": 16, "wall_time": 1.234, "iterations_total": 35, "t_neighbor": 1.0,
            "t_physics": 3.0, "t_rts": 0.0, "missed_neighbors": 0}
    lines = run_report(meta, audit=True)
    assert lines == ["solver pcisph-rts on 1000 fluid particles",
                     "simulated 0.5 s in 10 steps, 16 frames",
                     "wall time 1.23 s (3.50 iterations/step)",
                     "breakdown: neighbor 25.0%  physics 75.0%  rts 0.0%",
                     "missed neighbors: 0"]
    r = {"solver_a": "pcisph-const", "solver_b": "pcisph-rts", "speedup": 2.0,
         "iteration_ratio": 0.5, "work_ratio": 0.25, "com_deviation": 0.001,
         "com_deviation_frac": 0.0005, "frames_compared": 7}
    assert compare_report(r)[1] == "wall-clock speedup:  2.00x"
    assert compare_report(r)[4] == ("max COM deviation:   0.001000 m (0.050% of the domain "
                                    "diagonal, 7 frames)")
