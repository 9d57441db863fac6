"""The reference's own host-side tests, run unmodified against this package
(``rts_sph`` aliased to ``paper_2009_14514_b200`` by tests/ref_alias): scene
parsing and validation, stats I/O, kernel constants, frame I/O, compare and
the command line's configuration errors.  The device-backed tests of the
reference need a GPU and the reference tree together, which no single
machine here has; their equivalents are the -m gpu parity tests.

Skipped where the reference is not mounted (the GPU box)."""

import os
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))

CPU_SELECTION = [
    "test_scene.py",
    "test_stats.py",
    "test_kernels.py",
    "test_bench.py::test_frame_roundtrip_is_bitwise",
    "test_bench.py::test_frame_rejects_bad_magic",
    "test_bench.py::test_frame_rejects_truncation",
    "test_bench.py::test_frame_rejects_unknown_version",
    "test_bench.py::test_run_rejects_bad_arguments",
    "test_bench.py::test_compare_reports_known_ratios",
    "test_bench.py::test_compare_falls_back_to_compute_counts",
    "test_bench.py::test_compare_refuses_different_scenes",
    "test_bench.py::test_compare_requires_run_directories",
    "test_cli.py::test_bad_thread_env_is_a_config_error",
    "test_cli.py::test_bad_thread_count_is_a_config_error",
    "test_cli.py::test_missing_scene_exits_one",
    "test_cli.py::test_unknown_solver_exits_one",
    "test_cli.py::test_compare_rejects_non_run_directory",
]


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tree not mounted")
def test_reference_host_suite_passes_against_the_package(tmp_path):
    env = dict(os.environ, PYTHONPATH=os.path.join(HERE, "ref_alias"),
               PYTHONDONTWRITEBYTECODE="1")
    args = [sys.executable, "-m", "pytest", "-q", "-p", "rts_alias", "-p", "no:cacheprovider",
            "--rootdir", str(tmp_path)] + [os.path.join(REF_TESTS, t) for t in CPU_SELECTION]
    out = subprocess.run(args, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=600)
    tail = (out.stdout + out.stderr)[-3000:]
    assert out.returncode == 0, tail
    assert " passed" in out.stdout and "failed" not in out.stdout, tail
