"""bench.py's end-to-end path: the overlapped host round trip (results down on
the compute stream, the next step's inputs up on a side stream) must move
every byte both ways, in any chunking, and the solver must see exactly the
uploaded state in the next step."""

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("chunks", [0, 1, 3, 8])
def test_round_trip_moves_every_byte(chunks):
    import bench
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(chunks)
    n = 100_003  # not a multiple of any chunk count
    d_pos = torch.as_tensor(rng.normal(size=(n, 3)).astype(np.float32), device=dev)
    d_vel = torch.as_tensor(rng.normal(size=(n, 3)).astype(np.float32), device=dev)
    h_pos = torch.empty((n + 17, 3), dtype=torch.float32).pin_memory()
    h_vel = torch.empty((n + 17, 3), dtype=torch.float32).pin_memory()
    want_pos, want_vel = d_pos.cpu().clone(), d_vel.cpu().clone()
    rt = bench.HostRoundTrip(dev)
    rt.round_trip((d_pos, d_vel), (h_pos, h_vel), chunks=chunks)
    torch.cuda.synchronize()
    # the host holds the results, the device the uploaded copy of them
    assert torch.equal(h_pos[:n], want_pos) and torch.equal(h_vel[:n], want_vel)
    assert torch.equal(d_pos.cpu(), want_pos) and torch.equal(d_vel.cpu(), want_vel)
    # a host-side edit between steps reaches the device on the next upload
    h_pos[:n].mul_(2.0)
    rt.upload((d_pos, d_vel), (h_pos, h_vel))
    torch.cuda.synchronize()
    assert torch.equal(d_pos.cpu(), 2.0 * want_pos)


def test_host_owned_steps_match_device_resident_steps():
    """Three majors with the state round-tripping through pinned host memory
    after every major give the same state, bit for bit, as three majors that
    keep it on the device."""
    import bench
    from conftest import tiny_tank
    from paper_2009_14514_b200 import PcisphSolver
    dev = torch.device("cuda", 0)
    a = PcisphSolver(tiny_tank(), mode="rts", device=dev)
    b = PcisphSolver(tiny_tank(), mode="rts", device=dev)
    nf = a.n_fluid
    hp = torch.empty((nf, 3), dtype=torch.float32).pin_memory()
    hv = torch.empty((nf, 3), dtype=torch.float32).pin_memory()
    rt = bench.HostRoundTrip(dev)
    for k in range(3):
        a.advance()
        b.advance()
        rt.round_trip((b.pos[:nf], b.vel), (hp, hv))
    torch.cuda.synchronize()
    assert torch.equal(a.pos[:nf], b.pos[:nf]) and torch.equal(a.vel, b.vel)
    assert torch.equal(hp, a.pos[:nf].cpu()) and torch.equal(hv, a.vel.cpu())
