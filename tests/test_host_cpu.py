"""CPU: host-side logic of the drop-in and the C ABI of librtssph.so.

No kernel is launched here (no GPU in the build container): the library is
loaded, its exported symbols are checked against include/rts_sph.h, and the
ctypes structure layouts are checked against the C compiler's.
"""

import ctypes
import dataclasses
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, tiny_tank

from paper_2009_14514_b200 import (ConfigError, StepStats, load_scene, parse_scene_text,
                                   preset_scene, read_stats, seed_particles, write_stats)
from paper_2009_14514_b200 import _native as N

HEADER = os.path.join(ROOT, "include", "rts_sph.h")


# ---- C ABI ---------------------------------------------------------------

def _header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rts_\w+)\s*\(", text)))


def test_library_loads_and_exports_every_header_symbol():
    lib = N.load()
    assert lib.rts_abi_version() == N.ABI_VERSION
    names = _header_functions()
    assert len(names) > 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # every entry point the host binds is declared in the header
    assert set(N.SIGNATURES) <= set(names)


def _c_offsets(struct_name, fields):
    src = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', 'int main(void){']
    src.append(f'printf("%zu\\n", sizeof({struct_name}));')
    for f in fields:
        src.append(f'printf("%zu\\n", offsetof({struct_name}, {f}));')
    src.append("return 0;}")
    d = os.path.join(ROOT, "build")
    os.makedirs(d, exist_ok=True)
    c = os.path.join(d, f"abi_{struct_name}.c")
    exe = os.path.join(d, f"abi_{struct_name}")
    open(c, "w").write("\n".join(src))
    subprocess.run(["gcc", "-std=c11", "-o", exe, c], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    return [int(x) for x in out]


@pytest.mark.parametrize("cls,cname", [(N.RtsParams, "RtsParams"), (N.RtsCounters, "RtsCounters"),
                                       (N.RtsBuffers, "RtsBuffers"), (N.RtsControl, "RtsControl"),
                                       (N.RtsMinorStats, "RtsMinorStats")])
def test_struct_layouts_match_the_header(cls, cname):
    fields = [f[0] for f in cls._fields_]
    got = _c_offsets(cname, fields)
    assert got[0] == ctypes.sizeof(cls)
    for f, off in zip(fields, got[1:]):
        assert getattr(cls, f).offset == off, f


def test_solvers_refuse_to_run_without_cuda(monkeypatch):
    import torch

    from paper_2009_14514_b200 import PcisphSolver, WcsphSolver
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        WcsphSolver(tiny_tank())
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        PcisphSolver(tiny_tank(), device="cpu")


# ---- scene / stats / schedule host logic (reference pkg/tests) -----------------

def test_scene_parse_minimal_and_errors():
    sc = parse_scene_text("domain = 0 0 0  1 1 1\nspacing = 0.02\nfluid_box = 0 0 0  0.2 0.2 0.2\n")
    assert sc.domain_max == (1.0, 1.0, 1.0) and sc.spacing == 0.02
    with pytest.raises(ConfigError, match="line 3"):
        parse_scene_text("domain = 0 0 0 1 1 1\nspacing = 0.02\nbogus_key = 1\n")
    with pytest.raises(ConfigError, match="line 2"):
        parse_scene_text("domain = 0 0 0 1 1 1\nno equals sign here\n")
    with pytest.raises(ConfigError, match="line 1.*spacing"):
        parse_scene_text("spacing = fast\n")
    with pytest.raises(ConfigError, match="unknown preset"):
        parse_scene_text("preset = tsunami\n")
    with pytest.raises(ConfigError, match="missing required"):
        parse_scene_text("spacing = 0.02\n")


def test_scene_roundtrip_presets_and_derived():
    sc = tiny_tank()
    again = parse_scene_text(sc.to_config_text())
    assert again.scene_hash() == sc.scene_hash()
    assert again.base_dt("wcsph") == sc.base_dt("wcsph")
    p = parse_scene_text("preset = dam_break\nviscosity = 1e-5\n")
    assert p.name == "dam_break" and p.viscosity == 1e-5
    counts = {n: len(seed_particles(preset_scene(n))[0]) for n in
              ("dam_break", "double_dam_break", "block_drop", "corridor")}
    assert counts == {"dam_break": 8000, "double_dam_break": 30000, "block_drop": 13696,
                      "corridor": 7290}
    assert sc.particle_mass == pytest.approx(1000 * 0.02**3)
    assert sc.block_size("pcisph") == pytest.approx(0.044)
    assert sc.base_dt("wcsph") == 0.25 * (0.4 * 0.04 / 30.0)
    assert sc.base_dt("pcisph") == pytest.approx(0.0175 * 0.02)
    assert sc.const_dt() == pytest.approx(0.0083 * 0.02)
    b = sc.betas(4)
    assert np.isnan(b[0]) and np.isinf(b[1]) and b[2] == 0.4 and b[3] == pytest.approx(0.08)
    assert load_scene("corridor").name == "corridor"


def test_seeding_matches_reference_fixture_layout():
    g = np.load(os.path.join(ROOT, "tests", "golden", "grid_tiny.npz"))
    fluid, wall = seed_particles(tiny_tank())
    nf = int(g["n_fluid"])
    assert len(fluid) == nf
    # the fixture's wall rows are the reference's seeding, untouched by jitter
    assert np.array_equal(np.concatenate([fluid, wall])[nf:], g["pos"][nf:])


def test_stats_csv_roundtrip(tmp_path):
    rows = [StepStats(step=1, time=0.1, dt=0.1, n_compute=5, corrected=7, max_err=0.5),
            StepStats(step=2, time=0.2, dt=0.1, iters_r1=3, t_rts=1.25)]
    path = tmp_path / "s.csv"
    write_stats(path, rows)
    assert read_stats(path) == rows


def test_schedule_validation_and_controller():
    from paper_2009_14514_b200.pcisph import (DEFAULT_SCHEDULE, MajorStepController,
                                              validate_schedule)
    bad = list(DEFAULT_SCHEDULE)
    bad[1] = ((1, 2, 3), (1,), (1,))
    with pytest.raises(ConfigError, match="receives no iteration"):
        validate_schedule(tuple(bad))
    bad = list(DEFAULT_SCHEDULE)
    bad[0] = ((1, 2, 3, 4), (1,), (1,))
    with pytest.raises(ConfigError, match="fewer than 2 iterations on the first"):
        validate_schedule(tuple(bad))
    bad = list(DEFAULT_SCHEDULE)
    bad[1] = ((1, 2, 3, 4), (2,), (3,))
    with pytest.raises(ConfigError, match="region 1 receives fewer than 3"):
        validate_schedule(tuple(bad))
    ctl = MajorStepController(4, 4)
    ctl.note_major(True)
    assert (ctl.n_current, ctl.recovery_left) == (2, 10)
    for k in range(9):
        ctl.note_major(False)
    ctl.note_major(False)
    assert (ctl.n_current, ctl.recovery_left) == (4, 0)


def test_make_solver_rejects_unknown_names():
    from paper_2009_14514_b200 import make_solver
    with pytest.raises(ConfigError, match="unknown solver"):
        make_solver(tiny_tank(), "sph-turbo")


def test_row_mask_encoding_matches_schedule_rows():
    from paper_2009_14514_b200.pcisph import _row_mask
    assert _row_mask((1, 2, 3, 4)) == 0b11110
    assert _row_mask((1,)) == 0b10
    c = N.RtsControl()
    assert ctypes.sizeof(c) == ctypes.sizeof(N.RtsControl)
    assert dataclasses.is_dataclass(StepStats)


def test_comm_keyword_requires_the_default_group():
    """The ``comm`` keyword accepts only the default process group."""
    from paper_2009_14514_b200 import PcisphSolver, WcsphSolver
    from paper_2009_14514_b200.scene import Scene
    sc = Scene(domain_min=(0, 0, 0), domain_max=(0.2, 0.2, 0.2),
               fluid_boxes=(((0.0, 0.0, 0.0), (0.1, 0.1, 0.1)),), spacing=0.02)
    for cls in (WcsphSolver, PcisphSolver):
        with pytest.raises(ValueError, match="comm must be"):
            cls(sc, comm=object())


def test_schedule_validation_matches_the_reference_rules_on_random_schedules():
    """validate_schedule (table-driven rewrite) against the oracle's
    statement of pcisph.py:80-117: same verdict, same first message."""
    import random

    from oracle.sph import validate_schedule as reference_rules
    from paper_2009_14514_b200.pcisph import validate_schedule
    rng = random.Random(1)

    def verdict(f, sch):
        try:
            f(sch)
            return None
        except ConfigError as exc:
            return str(exc)

    legal = 0
    for _ in range(2000):
        sch = tuple(tuple(tuple(rng.sample(range(1, 6 if rng.random() < 0.05 else 5),
                                           rng.randint(1, 4)))
                          for _ in range(rng.randint(1, 4)))
                    for _ in range(rng.choice([2, 4])))
        a, b = verdict(validate_schedule, sch), verdict(reference_rules, sch)
        assert a == b, (sch, a, b)
        legal += a is None
    assert legal > 0


def test_nvtx_ranges_are_opt_in():
    """RTS_SPH_NVTX unset: the solvers' phase methods are the plain functions
    (no wrapper on the hot host path); set: each is wrapped in an NVTX range."""
    import subprocess
    import sys
    code = ("import paper_2009_14514_b200.pcisph as P, paper_2009_14514_b200.wcsph as W;"
            "print(hasattr(P.PcisphSolver.major_step, '__wrapped__'),"
            " hasattr(W.WcsphSolver.step, '__wrapped__'))")
    for flag, want in (("0", "False False"), ("1", "True True")):
        env = dict(os.environ, RTS_SPH_NVTX=flag)
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                             check=True, cwd=os.path.dirname(os.path.dirname(__file__)))
        assert out.stdout.strip() == want
