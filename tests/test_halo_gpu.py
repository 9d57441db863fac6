"""GPU: the x-slab exchange primitives of include/rts_sph.h.

``rts_halo_pack`` / ``rts_halo_unpack`` must move the listed rows of every
field bit for bit (fp32 rows, fp64 as two words, strided float4 lanes,
remapped storage rows, one received word stored twice) and reject malformed
specs; ``rts_ctl_publish`` / ``rts_ctl_fold`` must fold the per-rank
convergence scalars as MAX / rank-order SUM."""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _native():
    from paper_2009_14514_b200 import _native as N
    N.load()
    return N


def _spec(N, fields, msg_words):
    s = N.RtsHaloSpec()
    s.n_fields, s.msg_words = len(fields), msg_words
    s.row_words = sum(f[1] for f in fields)
    for k, (t, words, stride, remap, off) in enumerate(fields):
        s.f[k].ptr = t.data_ptr()
        s.f[k].remap = remap.data_ptr() if remap is not None else None
        s.f[k].words, s.f[k].stride, s.f[k].msg_off = words, stride, off
    return s


def test_pack_unpack_round_trip_bit_exact():
    N = _native()
    dev = torch.device("cuda:0")
    g = torch.Generator(device="cpu").manual_seed(7)
    n = 5000
    pos = torch.randn(n, 3, generator=g).to(dev)
    err = torch.randn(n, generator=g, dtype=torch.float64).to(dev)
    xs4 = torch.randn(n, 4, generator=g).to(dev)
    slot = torch.randperm(n, generator=g).to(torch.int32).to(dev)
    cpos = torch.randn(n, 4, generator=g).to(dev)
    rows = torch.sort(torch.randperm(n, generator=g)[:1234]).values.to(torch.int32).to(dev)
    pk = [(pos, 3, 3, None, 0), (err, 2, 2, None, 3), (xs4[:, 3:], 1, 4, None, 5)]
    msg = torch.empty((rows.numel(), 6), dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    N.call("rts_halo_pack", ctypes.byref(_spec(N, pk, 6)), rows.data_ptr(), rows.numel(),
           msg.data_ptr(), st)
    r = rows.long()
    m = msg.cpu()
    assert torch.equal(m[:, 0:3], pos[r].cpu().view(torch.int32))
    assert torch.equal(m[:, 3:5], err[r].cpu().view(torch.int32).reshape(-1, 2))
    assert torch.equal(m[:, 5], xs4[r, 3].cpu().view(torch.int32))

    # unpack into fresh storage; pos words also land in cpos at slot_of[row]
    pos2 = torch.zeros_like(pos)
    err2 = torch.zeros_like(err)
    xs42 = torch.zeros_like(xs4)
    cpos2 = cpos.clone()
    up = [(pos2, 3, 3, None, 0), (err2, 2, 2, None, 3), (xs42[:, 3:], 1, 4, None, 5),
          (cpos2, 3, 4, slot, 0)]
    N.call("rts_halo_unpack", ctypes.byref(_spec(N, up, 6)), rows.data_ptr(), rows.numel(),
           msg.data_ptr(), st)
    torch.cuda.synchronize()
    assert torch.equal(pos2[r], pos[r]) and torch.equal(err2[r], err[r])
    assert torch.equal(xs42[r, 3], xs4[r, 3])
    assert not pos2[~torch.isin(torch.arange(n, device=dev), r)].any()  # other rows untouched
    sl = slot[r].long()
    assert torch.equal(cpos2[sl, :3], pos[r]) and torch.equal(cpos2[sl, 3], cpos[sl, 3])
    keep = torch.ones(n, dtype=torch.bool, device=dev)
    keep[sl] = False
    assert torch.equal(cpos2[keep], cpos[keep])


def test_bad_spec_and_empty_rows():
    N = _native()
    dev = torch.device("cuda:0")
    a = torch.zeros(10, 3, device=dev)
    rows = torch.arange(4, dtype=torch.int32, device=dev)
    buf = torch.zeros(4, 3, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    bad = _spec(N, [(a, 3, 3, None, 1)], 3)  # field overruns the message row
    with pytest.raises(N.NativeError):
        N.call("rts_halo_pack", ctypes.byref(bad), rows.data_ptr(), 4, buf.data_ptr(), st)
    bad = _spec(N, [(a, 3, 2, None, 0)], 3)  # stride shorter than the row
    with pytest.raises(N.NativeError):
        N.call("rts_halo_unpack", ctypes.byref(bad), rows.data_ptr(), 4, buf.data_ptr(), st)
    ok = _spec(N, [(a, 3, 3, None, 0)], 3)
    N.call("rts_halo_pack", ctypes.byref(ok), rows.data_ptr(), 0, buf.data_ptr(), st)
    torch.cuda.synchronize()
    assert not buf.any()


def test_ctl_publish_fold():
    N = _native()
    dev = torch.device("cuda:0")
    size = ctypes.sizeof(N.RtsCounters)
    ctr = torch.zeros(size, dtype=torch.uint8, device=dev)
    host = N.RtsCounters()
    host.max_err, host.any_se, host.sum_rho, host.n_pred = 0.0125, 0, 1234.5, 77
    host.err_flags = 0
    ctr.copy_(torch.frombuffer(bytearray(bytes(host)), dtype=torch.uint8))
    b = N.RtsBuffers()
    b.ctr = ctr.data_ptr()
    W = N.CTL_WORDS
    out = torch.zeros(W, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    N.call("rts_ctl_publish", ctypes.byref(b), out.data_ptr(), st)
    assert out.cpu().tolist() == [0.0125, 0.0, 1234.5, 77.0, 0.0]
    gathered = torch.tensor([[0.0125, 0, 1234.5, 77, 0], [0.03, 1, 1e-3, 5, 0],
                             [0.01, 0, 7.25, 0, 0]], dtype=torch.float64, device=dev)
    N.call("rts_ctl_fold", ctypes.byref(b), gathered.data_ptr(), 3, st)
    torch.cuda.synchronize()
    c = N.RtsCounters.from_buffer_copy(bytes(ctr.cpu().numpy()))
    assert c.max_err == 0.03 and c.any_se == 1 and c.n_pred == 82 and c.err_flags == 0
    assert c.sum_rho == np.float64(1234.5) + np.float64(1e-3) + np.float64(7.25)
    with pytest.raises(N.NativeError):
        N.call("rts_ctl_fold", ctypes.byref(b), gathered.data_ptr(), 0, st)


def test_ctl_fold_spreads_a_rank_failure():
    """one rank's fatal flag or NaN error must reach every rank's
    k_control (same done / failed decision, no mismatched collectives)."""
    N = _native()
    dev = torch.device("cuda:0")
    ctr = torch.zeros(ctypes.sizeof(N.RtsCounters), dtype=torch.uint8, device=dev)
    b = N.RtsBuffers()
    b.ctr = ctr.data_ptr()
    st = torch.cuda.current_stream().cuda_stream
    nan = float("nan")
    gathered = torch.tensor([[0.01, 0, 1.0, 3, 0], [nan, 0, 1.0, 3, float(N.ERR_NONFINITE)]],
                            dtype=torch.float64, device=dev)
    N.call("rts_ctl_fold", ctypes.byref(b), gathered.data_ptr(), 2, st)
    torch.cuda.synchronize()
    c = N.RtsCounters.from_buffer_copy(bytes(ctr.cpu().numpy()))
    assert c.max_err != c.max_err  # NaN propagated
    assert c.err_flags & N.ERR_NONFINITE
