"""CPU: RTSF v1 frame I/O and the run comparison report (reference
pkg/tests/test_bench.py), on synthetic run directories."""

import json

import numpy as np
import pytest

from paper_2009_14514_b200 import ConfigError
from paper_2009_14514_b200.run import compare, frame_files, read_frame, write_frame


def test_frame_roundtrip_and_layout(tmp_path):
    pos = np.random.default_rng(0).random((17, 3)).astype(np.float32)
    reg = np.arange(17, dtype=np.uint8) % 5
    p = tmp_path / "frame_00003.bin"
    write_frame(p, 0.125, pos, reg)
    raw = p.read_bytes()
    assert raw[:4] == b"RTSF" and len(raw) == 20 + 17 * 13
    t, pos2, reg2 = read_frame(p)
    assert t == 0.125 and np.array_equal(pos2, pos) and np.array_equal(reg2, reg)
    assert frame_files(tmp_path) == [p]


def test_frame_errors(tmp_path):
    p = tmp_path / "f.bin"
    p.write_bytes(b"RT")
    with pytest.raises(ConfigError, match="truncated"):
        read_frame(p)
    write_frame(p, 0.0, np.zeros((2, 3)), np.zeros(2))
    raw = bytearray(p.read_bytes())
    raw[:4] = b"XXXX"
    p.write_bytes(bytes(raw))
    with pytest.raises(ConfigError, match="bad magic"):
        read_frame(p)
    write_frame(p, 0.0, np.zeros((2, 3)), np.zeros(2))
    p.write_bytes(p.read_bytes() + b"\0")
    with pytest.raises(ConfigError, match="expected"):
        read_frame(p)


def _fake_run(d, shift, wall, fps=10, n=5, scene_hash="h", corrected=100):
    d.mkdir()
    for k in range(n):
        pos = np.zeros((4, 3), dtype=np.float32) + shift * k
        write_frame(d / f"frame_{k:05d}.bin", k / fps, pos, np.ones(4))
    meta = {"solver": "x", "scene_hash": scene_hash, "fps": fps, "wall_time": wall,
            "iterations_total": 30, "corrected_total": corrected, "compute_total": 0,
            "domain_diagonal": 2.0}
    (d / "meta.json").write_text(json.dumps(meta))
    return d


def test_compare_reports_ratios_and_com_deviation(tmp_path):
    a = _fake_run(tmp_path / "a", 0.0, 2.0)
    b = _fake_run(tmp_path / "b", 0.01, 1.0, corrected=50)
    r = compare(a, b)
    assert r["speedup"] == 2.0 and r["work_ratio"] == 0.5 and r["iteration_ratio"] == 1.0
    assert r["com_deviation"] == pytest.approx(np.sqrt(3) * 0.04, rel=1e-6)
    assert r["com_deviation_frac"] == pytest.approx(r["com_deviation"] / 2.0)
    c = _fake_run(tmp_path / "c", 0.0, 1.0, scene_hash="other")
    with pytest.raises(ConfigError, match="different scenes"):
        compare(a, c)
    with pytest.raises(ConfigError, match="not a run directory"):
        compare(a, tmp_path)
