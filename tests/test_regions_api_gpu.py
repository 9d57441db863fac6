"""The public region-field functions (rts_sph.regions / grid helpers of the
reference) on the device, bit-exact against the oracle restatement on
random fields (the reference's test_regions.py strategy)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_region_functions_match_oracle(seed):
    from oracle import sph as O
    from paper_2009_14514_b200 import regions as R
    rng = np.random.default_rng(seed)
    dims = tuple(int(x) for x in rng.integers(3, 14, 3))
    n = int(np.prod(dims))
    occ = rng.random(n) < rng.uniform(0.2, 0.9)
    v = np.where(occ, rng.choice([0.0, 0.05, 0.3, 1.0, 3.0, 8.0], n) * rng.uniform(0.5, 1.5, n), 0.0)
    f = np.where(occ, rng.choice([0.0, 0.01, 0.1, 1.0, 10.0], n) * rng.uniform(0.5, 1.5, n), 0.0)
    kw = dict(dt_base=1e-3, block_size=0.04, particle_mass=0.008, sound_speed=30.0,
              lambda_v=0.4, lambda_f=0.25, alpha=1.0, betas=[np.inf, np.inf, 0.5, 0.25, 0.125],
              n_max=4)
    for sound in (True, False):
        got = R.assign_regions(v, f, occ, use_sound_criterion=sound, **kw)
        want = O.assign_regions(v, f, occ, use_sound_criterion=sound, **kw)
        assert np.array_equal(got, want)
    raw = O.assign_regions(v, f, occ, use_sound_criterion=False, **kw)
    sm, dropped = R.smooth_regions(raw, dims)
    sm_o, dropped_o = O.smooth_regions(raw, dims)
    assert np.array_equal(sm, sm_o) and np.array_equal(dropped, dropped_o)
    for layers in (1, 4):
        assert np.array_equal(R.expand_fast_regions(sm_o, dims, layers),
                              O.expand_fast_regions(sm_o, dims, layers))
    err = rng.random(n) < 0.05
    assert np.array_equal(R.derive_observed(sm_o, dims, err), O.derive_observed(sm_o, dims, err))
    mask = rng.random(dims) < 0.1
    for layers in (0, 1, 3):
        assert np.array_equal(R.dilate_mask(mask, layers), O.dilate_mask(mask, layers))
    fld = np.where(occ, raw, 127).astype(np.int8).reshape(dims)
    assert np.array_equal(R.neighbor_min(fld, 127), O.neighbor_min(fld, np.int8(127)))
