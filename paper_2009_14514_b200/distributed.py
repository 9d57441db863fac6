"""Multi-GPU RTS-SPH by x-slab decomposition.

One process per GPU (``torch.distributed``, NCCL over NVLink; gloo for the
1-GPU and CPU tests).  The padded block grid of the whole scene
(grid.py:223-244) is cut into x-slabs aligned to block faces; a rank owns
the fluid particles whose block column lies in its slab.

* ``DistributedWcsph`` / ``DistributedPcisph`` (the B200 ranks; also what
  ``WcsphSolver(..., comm=...)`` / ``PcisphSolver(..., comm=...)`` return):
  resident rank rows [owned | ghosts] in the solver arena.  At a step start
  (WCSPH) or major-step start (PCISPH) one exchange round moves migrants
  and a fresh ghost band (``rts_slab_classify``, ``rts_halo_pack`` /
  ``unpack``, ``rts_slab_holes``); the grid sort orders every block's fluid
  run by global id (``sort_key``), so each neighbour row and pair sum is the
  single-domain one.  WCSPH ghosts are recomputed redundantly and dropped
  (owned rows bit-identical to the single-domain run); PCISPH exchanges the
  inner ghost columns and folds the convergence scalars every correction
  iteration (``PcisphExchange``).  The cuts can be rebalanced by work.
* ``SlabWcsph``: the same slab protocol around any local step with the
  particle sets merged by global id -- the CPU tests run it with the oracle
  as the local step to check the protocol bit for bit.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from ._device import device_index, nvtx_range, raw_stream
from .errors import ConfigError, NumericalError
from .scene import Scene, seed_particles

# per-particle WCSPH state carried by ghosts and migrants, in pack order
WCSPH_FIELDS = (("pos", 3), ("vel", 3), ("acc", 3), ("acc_prev", 3), ("force", 3), ("rho", 1),
                ("pres", 1), ("dt_since", 1), ("dt_corr", 1), ("validity", 1), ("region", 1),
                ("compute", 1))
WCSPH_WIDTH = 1 + sum(w for _, w in WCSPH_FIELDS)  # + global id


@dataclass
class SlabPartition:
    """Block-aligned x-slabs of the padded grid of ``scene``."""

    origin_x: float
    inv_block: float
    nx: int
    world: int
    halo: int
    cuts: tuple = ()  # world + 1 column boundaries; empty = even split

    @classmethod
    def for_scene(cls, scene: Scene, mode: str, world: int, halo: int = 2,
                  balance: bool = True) -> "SlabPartition":
        pad = scene.boundary_layers * scene.spacing
        lo = scene.domain_min[0] - pad
        hi = scene.domain_max[0] + pad
        block = scene.block_size(mode)
        nx = max(1, int(math.ceil((hi - lo) / block - 1e-12)))
        part = cls(origin_x=lo, inv_block=1.0 / block, nx=nx, world=world, halo=halo)
        if balance and world > 1:
            # cut at equal fluid counts of the initial state (the RTS work
            # follows the particles; rebalancing at rebuilds is a next step)
            fluid, _ = seed_particles(scene)
            hist = np.bincount(part.block_x(fluid[:, 0]), minlength=nx).cumsum()
            total = hist[-1] if len(hist) else 0
            cuts = [0]
            w = max(1, halo)
            for r in range(1, world):
                c = int(np.searchsorted(hist, r * total / world, side="left")) + 1
                cuts.append(min(max(c, cuts[-1] + w), nx - w * (world - r)))
            cuts.append(nx)
            part.cuts = tuple(cuts)
        part.validate()
        return part

    def widths(self, cuts=None) -> list[int]:
        if cuts is None:
            return [b - a for a, b in (self.bounds(r) for r in range(self.world))]
        return [b - a for a, b in zip(cuts, cuts[1:])]

    def validate(self, cuts=None) -> None:
        """Every slab must hold at least ``halo`` block columns: a rank's ghost
        band comes from its immediate neighbours only, so a narrower slab
        would silently drop rows two ranks away."""
        for r, w in enumerate(self.widths(cuts)):
            if w < max(1, self.halo):
                raise ConfigError(
                    f"x-slab {r} is {w} block columns wide, narrower than the {self.halo}-column "
                    f"ghost band ({self.nx} columns for {self.world} ranks); use fewer ranks "
                    "or a longer domain")

    def rebalanced(self, weights) -> tuple:
        """Cuts at equal cumulative ``weights`` (per block column, summed over
        all ranks), each cut moved by less than the narrower slab next to it
        so that every particle's new owner is its old owner or a neighbour
        (rebalance at rebuilds from active-work counts)."""
        w = np.asarray(weights, dtype=np.float64).reshape(-1)
        cum = np.cumsum(w)
        total = cum[-1] if len(cum) else 0.0
        old = [self.bounds(r)[0] for r in range(self.world)] + [self.nx]
        cuts = [0]
        for r in range(1, self.world):
            want = int(np.searchsorted(cum, r * total / self.world, side="left")) + 1
            shift = min(old[r] - old[r - 1], old[r + 1] - old[r]) - 1
            c = min(max(want, old[r] - shift), old[r] + shift)
            c = min(max(c, cuts[-1] + 1), self.nx - (self.world - r))
            cuts.append(c)
        cuts.append(self.nx)
        if min(self.widths(cuts)) < max(1, self.halo):
            return tuple(old)  # no re-cut that keeps every slab as wide as the band
        return tuple(cuts)

    def bounds(self, rank: int) -> tuple[int, int]:
        """[first, last) block columns owned by ``rank``."""
        if self.cuts:
            return self.cuts[rank], self.cuts[rank + 1]
        base, rem = divmod(self.nx, self.world)
        lo = rank * base + min(rank, rem)
        return lo, lo + base + (1 if rank < rem else 0)

    def block_x(self, x) -> torch.Tensor | np.ndarray:
        """np.floor((x - origin) * inv_block), clipped (grid.py:248-250)."""
        if isinstance(x, torch.Tensor):
            c = torch.floor((x.double() - self.origin_x) * self.inv_block).long()
            return c.clamp(0, self.nx - 1)
        c = np.floor((np.asarray(x, dtype=np.float64) - self.origin_x) * self.inv_block)
        return np.clip(c.astype(np.int64), 0, self.nx - 1)

    def owner(self, bx):
        ranks = torch.arange(self.world) if isinstance(bx, torch.Tensor) else np.arange(self.world)
        highs = [self.bounds(r)[1] for r in range(self.world)]
        if isinstance(bx, torch.Tensor):
            h = torch.tensor(highs, device=bx.device)
            return torch.bucketize(bx, h, right=True).clamp(max=self.world - 1)
        return np.clip(np.searchsorted(np.asarray(highs), bx, side="right"), 0, self.world - 1)


def pack(state: dict, gid: torch.Tensor, fields=WCSPH_FIELDS) -> torch.Tensor:
    cols = [gid.double().reshape(-1, 1)]
    for name, w in fields:
        cols.append(state[name].double().reshape(-1, w))
    return torch.cat(cols, dim=1)


def unpack(rows: torch.Tensor, fields=WCSPH_FIELDS, dtypes=None) -> tuple[torch.Tensor, dict]:
    gid = rows[:, 0].long()
    out, c = {}, 1
    for name, w in fields:
        v = rows[:, c:c + w]
        out[name] = v if w > 1 else v.reshape(-1)
        c += w
    return gid, out


class Exchanger:
    """Paired neighbour send/recv of packed particle rows (counts first).

    ``device`` is where the rows live; ``comm_device`` where the transport
    wants them (the CUDA device for NCCL; "cpu" for gloo)."""

    def __init__(self, rank: int, world: int, device, comm_device=None):
        self.rank, self.world = rank, world
        self.compute_device = torch.device(device)
        self.device = torch.device(comm_device) if comm_device is not None else self.compute_device

    def _sendrecv(self, send: dict, width: int, dtype=torch.float64) -> list:
        """send: {peer: rows}; returns received row blocks from every peer
        that has a matching entry in its own ``send`` (symmetric pattern)."""
        peers = sorted(send)
        counts_out = {q: torch.tensor([send[q].shape[0]], dtype=torch.int64, device=self.device)
                      for q in peers}
        counts_in = {q: torch.zeros(1, dtype=torch.int64, device=self.device) for q in peers}
        ops = []
        for q in peers:
            ops.append(dist.P2POp(dist.isend, counts_out[q], q))
            ops.append(dist.P2POp(dist.irecv, counts_in[q], q))
        if ops:  # no peers (a single slab): nothing to exchange
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        bufs = {q: torch.empty((int(counts_in[q].item()), width), dtype=dtype,
                               device=self.device) for q in peers}
        ops = []
        for q in peers:
            if send[q].shape[0]:
                ops.append(dist.P2POp(dist.isend, send[q].to(self.device).contiguous(), q))
            if bufs[q].shape[0]:
                ops.append(dist.P2POp(dist.irecv, bufs[q], q))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        return [bufs[q].to(self.compute_device) for q in peers]

    def swap(self, send: dict, recv_rows: dict, width: int, dtype, out: dict | None = None) -> dict:
        """Exchange with known sizes (no count round): ``send`` {peer: rows},
        ``recv_rows`` {peer: expected row count}; returns {peer: rows}.  With
        ``out`` ({peer: preallocated rows} on the transport device) the rows
        are received in place."""
        bufs = out if out is not None else {
            q: torch.empty((recv_rows[q], width), dtype=dtype, device=self.device)
            for q in recv_rows}
        ops = []
        for q in sorted(send):
            if send[q].shape[0]:
                ops.append(dist.P2POp(dist.isend, send[q].to(self.device, dtype).contiguous(), q))
            if bufs[q].shape[0]:
                ops.append(dist.P2POp(dist.irecv, bufs[q], q))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        return {q: b.to(self.compute_device) for q, b in bufs.items()}

    def neighbours(self) -> list[int]:
        return [q for q in (self.rank - 1, self.rank + 1) if 0 <= q < self.world]


class SlabDriver:
    """Owns the rank's particles and runs the ghost / migrate protocol around
    a local step function ``local_step(fluid_state, gid) -> fluid_state``.

    ``SlabWcsph`` runs it around the oracle in the CPU tests (protocol
    checked bit for bit); the B200 ranks run the same ownership / band rules
    on resident rows (``_ResidentRank``) and use this class for the
    partition bounds and the transport.
    """

    def __init__(self, part: SlabPartition, rank: int, device, fields=WCSPH_FIELDS,
                 comm_device=None):
        self.part, self.rank, self.device, self.fields = part, rank, device, fields
        self.width = 1 + sum(w for _, w in fields)
        self.x = Exchanger(rank, part.world, device, comm_device)
        self.lo, self.hi = part.bounds(rank)

    def ghost_rows(self, gid, state) -> tuple[torch.Tensor, dict]:
        bx = self.part.block_x(state["pos"][:, 0])
        send = {}
        for q in self.x.neighbours():
            if q < self.rank:
                m = bx < self.lo + self.part.halo
            else:
                m = bx >= self.hi - self.part.halo
            idx = torch.nonzero(m).reshape(-1)
            send[q] = pack({k: v[idx] for k, v in state.items()}, gid[idx], self.fields)
        recv = self.x._sendrecv(send, self.width)
        rows = torch.cat(recv, 0) if recv else torch.zeros((0, self.width), dtype=torch.float64,
                                                           device=self.device)
        return unpack(rows, self.fields)

    def migrate(self, gid, state) -> tuple[torch.Tensor, dict]:
        bx = self.part.block_x(state["pos"][:, 0])
        own = self.part.owner(bx)
        keep = own == self.rank
        send = {}
        for q in self.x.neighbours():
            idx = torch.nonzero(own == q).reshape(-1)
            send[q] = pack({k: v[idx] for k, v in state.items()}, gid[idx], self.fields)
        far = (~keep) & torch.isin(own, torch.tensor(self.x.neighbours() or [-1],
                                                     device=own.device), invert=True)
        if bool(far.any()):
            raise RuntimeError("a particle crossed more than one slab in one step")
        recv = self.x._sendrecv(send, self.width)
        # kept rows stay in their dtypes and their (global-id) order; only
        # arrivals force a merge by global id
        leaving = not bool(keep.all())
        if leaving:
            kidx = torch.nonzero(keep).reshape(-1)
            gid = gid[kidx]
            state = {k: v[kidx] for k, v in state.items()}
        rows = torch.cat(recv, 0) if recv else None
        if rows is None or rows.shape[0] == 0:
            return gid, state
        rgid, rstate = unpack(rows, self.fields)
        allg = torch.cat([gid, rgid.to(gid.dtype)])
        order = torch.argsort(allg)
        out = {k: torch.cat([v, rstate[k].to(v.dtype).reshape((-1,) + v.shape[1:])])[order]
               for k, v in state.items()}
        return allg[order], out

    def merged(self, gid, state, ggid, gstate):
        """Owned + ghosts sorted by global id (the single-domain order)."""
        allg = torch.cat([gid, ggid])
        order = torch.argsort(allg)
        merged = {k: torch.cat([state[k].to(gstate[k].dtype), gstate[k]])[order] for k in state}
        is_owned = torch.cat([torch.ones_like(gid, dtype=torch.bool),
                              torch.zeros_like(ggid, dtype=torch.bool)])[order]
        return allg[order], merged, is_owned


def initial_ownership(scene: Scene, part: SlabPartition, rank: int):
    """Global ids and positions of the fluid particles ``rank`` owns at t=0,
    and the wall samples it needs (slab + halo columns), as float64 numpy."""
    fluid, wall = seed_particles(scene)
    bx = part.block_x(fluid[:, 0])
    gid = np.flatnonzero(part.owner(bx) == rank)
    lo, hi = part.bounds(rank)
    wb = part.block_x(wall[:, 0]) if len(wall) else np.zeros(0, dtype=np.int64)
    wsel = np.flatnonzero((wb >= lo - part.halo - 1) & (wb < hi + part.halo + 1))
    return gid, fluid, wall, wsel


class SlabWcsph:
    """The x-slab protocol of RTS-WCSPH around any local step (the CPU tests
    plug the oracle in): ``step()`` = ghost exchange, one local step on
    owned + ghosts merged by global id, extraction of the owned rows,
    migration.  The B200 ranks run the same protocol on resident rows
    (``DistributedWcsph``)."""

    def __init__(self, scene: Scene, local, mode: str = "rts", device=None, halo: int = 2,
                 jitter=None, comm_device=None, velocity=None):
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.part = SlabPartition.for_scene(scene, "wcsph", self.world, halo)
        gid, fluid, wall, wsel = initial_ownership(scene, self.part, self.rank)
        if jitter is not None:
            fluid = (fluid + jitter).astype(np.float32).astype(np.float64)
        if comm_device is None and dist.get_backend() == "gloo":
            comm_device = "cpu"
        self.driver = SlabDriver(self.part, self.rank, self.device, comm_device=comm_device)
        self.n_global = len(fluid)
        self.solver = local
        self.solver._set_local_particles(None, wall[wsel], capacity=None, init=True)
        self.gid = torch.as_tensor(gid, device=self.device)
        fl = torch.as_tensor(fluid[gid].astype(np.float32), device=self.device)
        self.state = self.solver._fresh_state(fl)
        if velocity is not None:  # (n_global, 3) initial velocities by global id
            self.state["vel"] = torch.as_tensor(np.asarray(velocity)[gid], device=self.device,
                                                dtype=self.state["vel"].dtype)
        self.sim_time = 0.0
        self.step_index = 0

    @property
    def n_owned(self) -> int:
        return int(self.gid.numel())

    def step(self):
        ggid, gstate = self.driver.ghost_rows(self.gid, self.state)
        allg, merged, owned = self.driver.merged(self.gid, self.state, ggid, gstate)
        self.solver._set_local_particles(merged, None)
        st = self.solver.step()
        out = self.solver._get_local_state()
        idx = torch.nonzero(owned).reshape(-1)
        state = {k: v[idx] for k, v in out.items()}
        st.n_compute = int(state["compute"].sum())  # owned particles only
        self.gid, self.state = self.driver.migrate(allg[idx], state)
        self.state = self.solver._cast_state(self.state)
        self.sim_time += st.dt
        self.step_index += 1
        return st


# ---------------------------------------------------------------------------
# RTS-PCISPH over x-slabs
# ---------------------------------------------------------------------------

class HaloChannel:
    """One fixed-row exchange phase of a major step, native end to end:
    ``rts_halo_pack`` of every peer's send rows into one word buffer, a
    grouped send/recv of the per-peer slices (NCCL: stream-ordered, no host
    synchronisation), ``rts_halo_unpack`` of the received rows.

    ``pack`` / ``unpack``: ``(tensor, words, stride, remap, msg_off)`` in
    32-bit words (fp64 = 2 words, bit copies).  Unpack fields may share
    message words, so one received word can be stored in two places."""

    def __init__(self, xch: "Exchanger", send_idx: dict, recv_idx: dict, pack, unpack=None):
        from . import _native as N
        self.N, self.x = N, xch
        self.peers = sorted(send_idx)
        dev = xch.compute_device

        def rows(d):
            if not self.peers:
                return torch.zeros(0, dtype=torch.int32, device=dev)
            return torch.cat([d[q].reshape(-1) for q in self.peers]).to(torch.int32).contiguous()

        self.send_rows, self.recv_rows = rows(send_idx), rows(recv_idx)
        self.n_send = [int(send_idx[q].numel()) for q in self.peers]
        self.n_recv = [int(recv_idx[q].numel()) for q in self.peers]
        self.msg_words = max(f[4] + f[1] for f in pack)
        self.pack_spec = self._spec(pack)
        self.unpack_spec = self._spec(unpack or pack)
        self.send_buf = torch.empty((sum(self.n_send), self.msg_words), dtype=torch.int32,
                                    device=dev)
        self.recv_buf = torch.empty((sum(self.n_recv), self.msg_words), dtype=torch.int32,
                                    device=dev)
        self.recv_views, b = {}, 0
        for q, nr in zip(self.peers, self.n_recv):
            self.recv_views[q] = self.recv_buf[b:b + nr]
            b += nr

    def _spec(self, fields):
        N = self.N
        if not 1 <= len(fields) <= N.HALO_MAX_FIELDS:
            raise ValueError(f"{len(fields)} halo fields (1..{N.HALO_MAX_FIELDS})")
        spec = N.RtsHaloSpec()
        spec.n_fields, spec.msg_words = len(fields), self.msg_words
        spec.row_words = sum(f[1] for f in fields)
        for k, (t, words, stride, remap, off) in enumerate(fields):
            f = spec.f[k]
            f.ptr = t.data_ptr()
            f.remap = remap.data_ptr() if remap is not None else None
            f.words, f.stride, f.msg_off = words, stride, off
        return spec

    def run(self) -> None:
        if not self.peers:
            return
        N = self.N
        st = raw_stream(device_index(self.x.compute_device))
        N.call("rts_halo_pack", ctypes.byref(self.pack_spec), self.send_rows.data_ptr(),
               self.send_rows.numel(), self.send_buf.data_ptr(), st)
        send, a = {}, 0
        for q, ns in zip(self.peers, self.n_send):
            send[q] = self.send_buf[a:a + ns]
            a += ns
        direct = self.x.device == self.x.compute_device  # NCCL: receive in place
        got = self.x.swap(send, dict(zip(self.peers, self.n_recv)), self.msg_words, torch.int32,
                          out=self.recv_views if direct else None)
        if not self.recv_rows.numel():
            return
        if not direct:
            b = 0
            for q, nr in zip(self.peers, self.n_recv):
                self.recv_buf[b:b + nr].copy_(got[q])
                b += nr
        N.call("rts_halo_unpack", ctypes.byref(self.unpack_spec), self.recv_rows.data_ptr(),
               self.recv_rows.numel(), self.recv_buf.data_ptr(), st)


class PcisphExchange:
    """Ghost refreshes inside a major step (hooks called by PcisphSolver's
    host-driven loop).  Only the two inner ghost columns on each side are
    neighbours of owned particles (two layers of 2.2s blocks cover the
    region-1 two-layer search); deeper ghosts exist for the major-start
    level fields only.  Per correction iteration: x* after the motion pass,
    p / err / rho* after the density pass, then the convergence scalars
    (max err, sum rho*, any S_e, |pred|) of every rank all-gathered and
    folded on the device in rank order -- the exchange steps of SURVEY.md
    section 8e.  Per minor step: pos / vel / f_ext / f_p after the
    integrator (next refresh, mid-major marking).  Every phase is one native
    pack, one grouped send/recv and one native unpack (``HaloChannel``)."""

    def __init__(self, driver: "SlabDriver", send_idx: dict, recv_idx: dict):
        self.x = driver.x
        self.send_idx, self.recv_idx = send_idx, recv_idx
        self.peers = sorted(send_idx)
        self._ch = None
        from . import _native as N
        self.N_CTL = N.CTL_WORDS

    def _channels(self, s) -> dict:
        if self._ch is None:
            A = s.arena
            xs, err, rho = A["xs"], A["err"], A["rho"]
            xw = xs.view(torch.int32)  # 8 words per row: fp64 x* (6), fp64 p (2)
            pos, vel, fe, fp = A["pos"], A["vel"], A["force"], A["f_p"]
            ch = lambda pk, up=None: HaloChannel(self.x, self.send_idx, self.recv_idx, pk, up)
            # the fp64 p of the xs rows (the pair passes read it; pres is its
            # fp32 mirror, not needed on ghosts), err, rho*
            dens = [(xw[:, 6:], 2, 8, None, 0), (err, 2, 2, None, 2), (rho, 1, 1, None, 4)]
            move = [(pos, 3, 3, None, 0), (vel, 3, 3, None, 3), (fe, 3, 3, None, 6),
                    (fp, 3, 3, None, 9)]
            self._ch = {
                "motion": ch([(xw, 8, 8, None, 0)]),  # x* and p (zeroed / restored)
                "density": ch(dens),
                # pos also refreshes the candidate copy at the row's CSR slot
                "integrate": ch(move, move + [(A["cpos"], 3, 4, A["slot_of"], 0)]),
            }
            dev = self.x.compute_device
            W = self.N_CTL
            self._pub = torch.zeros(W, dtype=torch.float64, device=dev)
            self._gath = torch.zeros((self.x.world, W), dtype=torch.float64, device=dev)
        return self._ch

    def after_motion(self, s) -> None:
        self._channels(s)["motion"].run()

    def after_density(self, s) -> None:
        self._channels(s)["density"].run()

    def reduce(self, s) -> None:
        from . import _native as N
        self._channels(s)
        st = raw_stream(device_index(self.x.compute_device))
        N.call("rts_ctl_publish", s.arena.buf, self._pub.data_ptr(), st)
        if self.x.device == self.x.compute_device:  # NCCL: gather in place, stream-ordered
            dist.all_gather_into_tensor(self._gath, self._pub)
        else:
            pub = self._pub.to(self.x.device)
            parts = [torch.empty_like(pub) for _ in range(self.x.world)]
            dist.all_gather(parts, pub)
            self._gath.copy_(torch.stack(parts))
        N.call("rts_ctl_fold", s.arena.buf, self._gath.data_ptr(), self.x.world, st)

    def after_integrate(self, s) -> None:
        self._channels(s)["integrate"].run()


class RankRows:
    """Full-row moves of a rank's resident fluid rows (pos, every state
    field of the solver, and the global id kept in ``sort_key``) through
    ``rts_halo_pack`` / ``rts_halo_unpack``: migrants out, arrivals and
    ghosts in, hole filling -- no per-field host indexing, no re-sort."""

    def __init__(self, solver):
        self.s = solver
        self._key = None

    @staticmethod
    def _layout(t: torch.Tensor, width: int) -> tuple[int, int, int]:
        """(elements per row, element stride, element bytes) of a field."""
        if t.element_size() == 8:
            return 2 * width, 2 * width, 4
        if t.element_size() == 4:
            return width, width, 4
        if t.element_size() == 1:
            return width, width, 1
        raise TypeError(f"unsupported field dtype {t.dtype}")

    def spec(self):
        from . import _native as N
        s, A = self.s, self.s.arena
        names = [("pos", 3)] + [(arena, w) for _, arena, w, *_ in s._FIELDS] + [("sort_key", 1)]
        key = tuple(A[n].data_ptr() for n, _ in names)
        if key != self._key:
            fields, off = [], 0
            for name, w in names:
                words, stride, esize = self._layout(A[name], w)
                fields.append((A[name], words, stride, esize, off))
                off += words
            sp = N.RtsHaloSpec()
            sp.n_fields, sp.row_words, sp.msg_words = len(fields), off, off
            for k, (t, words, stride, esize, o) in enumerate(fields):
                f = sp.f[k]
                f.ptr, f.remap = t.data_ptr(), None
                f.words, f.stride, f.msg_off, f.esize = words, stride, o, esize
            self._spec, self._words, self._key = sp, off, key
        return self._spec

    @property
    def words(self) -> int:
        self.spec()
        return self._words

    def pack(self, rows: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        from . import _native as N
        sp = self.spec()
        if out is None:
            out = torch.empty((rows.numel(), self.words), dtype=torch.int32, device=rows.device)
        if rows.numel():
            r = rows.to(torch.int32).contiguous()
            N.call("rts_halo_pack", ctypes.byref(sp), r.data_ptr(), r.numel(), out.data_ptr(),
                   raw_stream(device_index(rows.device)))
        return out

    def unpack(self, rows: torch.Tensor, msg: torch.Tensor) -> None:
        from . import _native as N
        if not rows.numel():
            return
        sp = self.spec()
        r = rows.to(torch.int32).contiguous()
        m = msg.to(rows.device, torch.int32).contiguous()
        N.call("rts_halo_unpack", ctypes.byref(sp), r.data_ptr(), r.numel(), m.data_ptr(),
               raw_stream(device_index(rows.device)))


class _ResidentRank:
    """Resident rank rows: the solver's fluid rows are [owned | ghosts].
    Migrants leave by hole filling; arrivals and the ghost band are unpacked
    behind the owned rows -- each phase one native pack, one grouped
    send/recv (count first) and one native unpack.  Row order is free: the
    grid sort orders every block's fluid run by global id (``sort_key``),
    so every neighbour row and pair sum is the single-domain one."""

    def _init_rows(self, gid: np.ndarray, state: dict, halo: int) -> None:
        s = self.solver
        fx = state["pos"][:, 0].double().cpu().numpy()
        bx = self.part.block_x(fx) if len(gid) else np.zeros(0, dtype=np.int64)
        lo, hi = self.driver.lo, self.driver.hi
        band = int(((bx < lo + halo) | (bx >= hi - halo)).sum())
        s._set_local_particles(state, None, capacity=int(1.25 * (len(gid) + 2 * band)) + 4096)
        self._alloc_key()
        s.arena["sort_key"][:len(gid)] = torch.as_tensor(gid, dtype=torch.int32, device=self.device)
        self.rows = RankRows(s)
        self.n_own = len(gid)

    # -- work rebalancing ----------------------------------------
    rebalance_every = 0   # majors (PCISPH) / steps (WCSPH) between checks; 0 = off
    rebalance_tol = 1.10  # rebalance when the busiest rank has > tol x the mean work

    def _work_weights(self, n: int) -> torch.Tensor:
        """Relative work of the owned rows for one major step / step."""
        return torch.ones(n, dtype=torch.float64, device=self.device)

    def rebalance(self) -> bool:
        """Move the slab cuts to equal work: per-column work of the owned rows,
        all-reduced; new cuts where the busiest rank exceeds ``rebalance_tol``
        times the mean.  The rows follow by the next exchange (two rounds:
        arrivals may land deeper than one column); the wall samples of the
        new slab + halo are re-selected.  Returns whether the cuts moved."""
        s, n, part = self.solver, self.n_own, self.part
        bx = part.block_x(s.arena["pos"][:n, 0])
        hist = torch.zeros(part.nx, dtype=torch.float64, device=self.device)
        hist.index_add_(0, bx, self._work_weights(n))
        h = hist.to(self.x.device)
        dist.all_reduce(h)
        h = h.cpu().numpy()
        per_rank = [h[a:b].sum() for a, b in (part.bounds(r) for r in range(self.world))]
        mean = sum(per_rank) / self.world
        if self.world < 2 or mean <= 0 or max(per_rank) <= self.rebalance_tol * mean:
            return False
        cuts = part.rebalanced(h)
        if cuts == tuple(part.bounds(r)[0] for r in range(self.world)) + (part.nx,):
            return False
        part.cuts = cuts
        self.driver.lo, self.driver.hi = part.bounds(self.rank)
        self._one_round = None  # re-derived; this exchange takes two rounds
        self._force_two_rounds = True
        lo, hi, h2 = self.driver.lo, self.driver.hi, part.halo + 1
        wsel = np.flatnonzero((self._wall_bx >= lo - h2) & (self._wall_bx < hi + h2))
        keep = {k: v.clone() for k, v in s._get_local_state().items()}
        key = s.arena["sort_key"][:s.n_fluid].clone()
        s._set_local_particles(keep, self._wall_all[wsel], capacity=s._cap)
        self._alloc_key()
        s.arena["sort_key"][:key.numel()] = key
        self.rows._key = None
        s._resize_fluid(self.n_own, s.n_fluid - self.n_own)
        return True

    def _keep_walls(self, wall: np.ndarray) -> None:
        self._wall_all = wall
        self._wall_bx = (self.part.block_x(wall[:, 0]) if len(wall)
                         else np.zeros(0, dtype=np.int64))

    def _maybe_rebalance(self, count: int) -> None:
        if self.rebalance_every and count and count % self.rebalance_every == 0:
            self.rebalance()

    def _alloc_key(self) -> None:
        A = self.solver.arena
        cap = self.solver._cap
        if "sort_key" not in A.t or A["sort_key"].numel() < cap:
            old = A.t.get("sort_key")
            k = A.alloc("sort_key", (cap,), torch.int32, 0)
            if old is not None:
                k[:old.numel()] = old

    @property
    def gid(self) -> torch.Tensor:
        return self.solver.arena["sort_key"][:self.n_own].long()

    @property
    def state(self) -> dict:
        """Views of the owned rows (writable in place)."""
        out = self.solver._get_local_state()
        return {k: v[:self.n_own] for k, v in out.items()}

    @property
    def n_owned(self) -> int:
        return self.n_own

    # reference-facing view of a rank (WcsphSolver / PcisphSolver attributes
    # callers read, bench.py:129-166): the owned rows
    @property
    def n_fluid(self) -> int:
        return self.n_own

    @property
    def pos(self) -> torch.Tensor:
        return self.solver.arena["pos"][:self.n_own]

    @property
    def vel(self) -> torch.Tensor:
        return self.solver.arena["vel"][:self.n_own]

    @property
    def missed_neighbors_total(self) -> int:
        return int(getattr(self.solver, "missed_neighbors_total", 0))

    def particle_regions(self) -> torch.Tensor:
        return self.solver.particle_regions()[:self.n_own]

    def _resize(self, nf: int, n_ghost: int) -> None:
        s = self.solver
        if nf > s._cap:  # grow, keeping the current rows (rare)
            keep = {k: v.clone() for k, v in s._get_local_state().items()}
            key = s.arena["sort_key"][:s.n_fluid].clone()
            s._set_local_particles(keep, None, capacity=int(1.25 * nf) + 4096)
            self._alloc_key()
            s.arena["sort_key"][:key.numel()] = key
            self.rows._key = None
        s._resize_fluid(nf, n_ghost)

    def _exchange_rows(self, send: dict) -> torch.Tensor:
        """Rows packed per peer -> the received rows, concatenated in peer order."""
        packed = {q: self.rows.pack(idx) for q, idx in send.items()}
        recv = self.x._sendrecv(packed, self.rows.words, torch.int32)
        recv = [r for r in recv if r.shape[0]]
        if not recv:
            return torch.zeros((0, self.rows.words), dtype=torch.int32, device=self.device)
        return torch.cat(recv) if len(recv) > 1 else recv[0]

    def _single_round(self) -> bool:
        """Migration and the ghost band fit one exchange round when every slab
        is wider than halo + 1 columns: an arrival (it moved less than one
        column) can then never land in the band next to the *other*
        neighbour, so a rank's post-migration band = its kept band rows plus
        the migrants it just received from that same neighbour -- which the
        neighbour keeps as ghosts itself (lists 4 / 5 of rts_slab_classify)."""
        if getattr(self, "_one_round", None) is None:
            widths = [b - a for a, b in (self.part.bounds(r) for r in range(self.world))]
            self._one_round = min(widths) > self.part.halo + 1
        return self._one_round

    @nvtx_range("rts_slab.exchange")
    def _exchange(self) -> None:
        """Migration + fresh ghost band (one round when ``_single_round``)."""
        if getattr(self, "_force_two_rounds", False) or not self._single_round():
            self._force_two_rounds = False
            self._migrate()
            self._ghosts()
            return
        from . import _native as N
        s, n, dev = self.solver, self.n_own, self.device
        st = torch.cuda.current_stream(dev).cuda_stream
        part, r = self.part, self.rank
        lo, hi = part.bounds(r)
        g = N.RtsSlabGeom(origin_x=part.origin_x, inv_block=part.inv_block, nx=part.nx, lo=lo,
                          hi=hi, halo=part.halo, has_left=int(r > 0),
                          has_right=int(r < self.world - 1),
                          left_lo=part.bounds(r - 1)[0] if r > 0 else lo,
                          right_hi=part.bounds(r + 1)[1] if r < self.world - 1 else hi)
        ls = max(n, 1)
        lists = torch.empty((6, ls), dtype=torch.int32, device=dev)
        leave = torch.empty(ls, dtype=torch.uint8, device=dev)
        counts = torch.empty(8, dtype=torch.int32, device=dev)
        N.call("rts_slab_classify", ctypes.byref(g), s.arena["pos"].data_ptr(), n,
               lists.data_ptr(), ls, leave.data_ptr(), counts.data_ptr(), st)
        c = counts.tolist()  # one host sync: the message sizes
        self._agree_or_raise(c[6], "a particle crossed more than one slab in one step")
        W = self.rows.words
        send, keepg = {}, []
        for q, (mig, band, selfg) in ((r - 1, (0, 2, 4)), (r + 1, (1, 3, 5))):
            if not 0 <= q < self.world:
                continue
            nm, nb = c[mig], c[band]
            buf = torch.empty((nm + nb, W), dtype=torch.int32, device=dev)
            self.rows.pack(lists[mig, :nm], buf[:nm])
            self.rows.pack(lists[band, :nb], buf[nm:])
            send[q] = (nm, buf)
            keepg.append(lists[selfg, :c[selfg]])
        selfg = self.rows.pack(torch.cat(keepg)) if keepg else None
        recv = self._sendrecv_split(send)
        n_leave = c[0] + c[1]
        n_keep = n - n_leave
        if n_leave:  # fill the holes below n_keep with the kept rows above it
            plan = torch.empty((2, n_leave), dtype=torch.int32, device=dev)
            N.call("rts_slab_holes", leave.data_ptr(), n, n_keep, n_leave, plan[0].data_ptr(),
                   plan[1].data_ptr(), counts.data_ptr(), st)
            self.rows.unpack(plan[0], self.rows.pack(plan[1]))
        arr = [m[:k] for k, m in recv]
        gh = [m[k:] for k, m in recv] + ([selfg] if selfg is not None else [])
        arr = torch.cat(arr) if arr else torch.zeros((0, W), dtype=torch.int32, device=dev)
        gh = torch.cat(gh) if gh else torch.zeros((0, W), dtype=torch.int32, device=dev)
        n_own = n_keep + arr.shape[0]
        self._resize(n_own + gh.shape[0], gh.shape[0])
        self.rows.unpack(torch.arange(n_keep, n_own, device=dev), arr)
        self.rows.unpack(torch.arange(n_own, n_own + gh.shape[0], device=dev), gh)
        self.n_own = n_own

    def _agree_or_raise(self, bad: int, msg: str) -> None:
        """Raise on every rank when ``bad`` is non-zero on any of them (a
        rank-local raise would leave its peers waiting in the next exchange)."""
        t = torch.tensor([float(bad)], dtype=torch.float64, device=self.x.device)
        dist.all_reduce(t)
        if float(t.item()):
            raise RuntimeError(msg if bad else f"another x-slab rank: {msg}")

    def _sendrecv_split(self, send: dict) -> list:
        """send {peer: (n_first, rows)} -> [(n_first, rows)] per peer: the row
        counts of both parts travel first (one int64 pair per peer)."""
        x, dev = self.x, self.x.device
        peers = sorted(send)
        cout = {q: torch.tensor([send[q][0], send[q][1].shape[0]], dtype=torch.int64, device=dev)
                for q in peers}
        cin = {q: torch.zeros(2, dtype=torch.int64, device=dev) for q in peers}
        ops = []
        for q in peers:
            ops += [dist.P2POp(dist.isend, cout[q], q), dist.P2POp(dist.irecv, cin[q], q)]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        sizes = {q: cin[q].tolist() for q in peers}
        bufs = {q: torch.empty((sizes[q][1], self.rows.words), dtype=torch.int32, device=dev)
                for q in peers}
        ops = []
        for q in peers:
            if send[q][1].shape[0]:
                ops.append(dist.P2POp(dist.isend, send[q][1].to(dev).contiguous(), q))
            if bufs[q].shape[0]:
                ops.append(dist.P2POp(dist.irecv, bufs[q], q))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return [(sizes[q][0], bufs[q].to(self.device)) for q in peers]

    def _migrate(self) -> None:
        """Owned rows whose block column left the slab go to the neighbour."""
        s, n = self.solver, self.n_own
        own = self.part.owner(self.part.block_x(s.arena["pos"][:n, 0]))
        leave = own != self.rank
        far = (own - self.rank).abs() > 1
        n_far, n_leave = torch.stack([far.sum(), leave.sum()]).tolist()  # one host sync
        self._agree_or_raise(n_far, "a particle crossed more than one slab in one step")
        arr = self._exchange_rows({q: torch.nonzero(own == q).reshape(-1)
                                   for q in self.x.neighbours()})
        n_keep = n - n_leave
        if n_leave:  # fill the holes below n_keep with the kept rows above it
            holes = torch.nonzero(leave[:n_keep]).reshape(-1)
            fill = torch.nonzero(~leave[n_keep:]).reshape(-1) + n_keep
            if holes.numel():
                self.rows.unpack(holes, self.rows.pack(fill))
        self._resize(n_keep + arr.shape[0], 0)
        self.rows.unpack(torch.arange(n_keep, n_keep + arr.shape[0], device=self.device), arr)
        self.n_own = n_keep + arr.shape[0]

    def _ghosts(self) -> None:
        """Owned rows in the ``halo`` block columns next to each neighbour are
        copied to it; the received ones become this rank's ghost rows."""
        s, n = self.solver, self.n_own
        bx = self.part.block_x(s.arena["pos"][:n, 0])
        lo, hi, h = self.driver.lo, self.driver.hi, self.part.halo
        send = {}
        for q in self.x.neighbours():
            m = bx < lo + h if q < self.rank else bx >= hi - h
            send[q] = torch.nonzero(m).reshape(-1)
        g = self._exchange_rows(send)
        self._resize(n + g.shape[0], g.shape[0])
        self.rows.unpack(torch.arange(n, n + g.shape[0], device=self.device), g)


class DistributedWcsph(_ResidentRank):
    """RTS-WCSPH over x-slabs on the B200: ``step()`` = migration and a fresh
    2-column ghost band on resident rows (the first band's densities need
    the second band's positions, its smoothed levels the second band's raw
    levels), then one B200 step on owned + ghosts; the ghosts are recomputed
    redundantly and dropped, so there is no exchange inside the step.  Owned
    results are bit-identical to the single-domain run.  The baseline's CFL
    bound is an all-reduce MAX of |F|."""

    def __init__(self, scene: Scene, mode: str = "rts", device=None, halo: int = 2,
                 jitter=None, comm_device=None, velocity=None, balance: bool = True,
                 rebalance_every: int = 0, **kw):
        from .wcsph import WcsphSolver
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.part = SlabPartition.for_scene(scene, "wcsph", self.world, halo, balance)
        self.rebalance_every = rebalance_every
        gid, fluid, wall, wsel = initial_ownership(scene, self.part, self.rank)
        self._keep_walls(wall)
        if jitter is not None:
            fluid = (fluid + jitter).astype(np.float32).astype(np.float64)
        if comm_device is None and dist.get_backend() == "gloo":
            comm_device = "cpu"
        self.driver = SlabDriver(self.part, self.rank, self.device, comm_device=comm_device)
        self.x = self.driver.x
        self.n_global = len(fluid)
        # graphs off: the particle count changes every step
        s = self.solver = WcsphSolver(scene, mode=mode, device=self.device, use_graphs=False, **kw)
        s._set_local_particles(None, wall[wsel], capacity=None, init=True)
        s._reduce_max = self._all_max
        fl = torch.as_tensor(fluid[gid].astype(np.float32), device=self.device)
        st = s._fresh_state(fl)
        if velocity is not None:  # (n_global, 3) initial velocities by global id
            st["vel"] = torch.as_tensor(np.asarray(velocity)[gid], device=self.device,
                                        dtype=st["vel"].dtype)
        self._init_rows(gid, st, halo)
        self.sim_time = 0.0
        self.step_index = 0

    def _work_weights(self, n: int) -> torch.Tensor:
        """Region n is active every 2^(n-1) base steps (wcsph.py:237-266)."""
        reg = self.solver.arena["region"][:n].double().clamp(min=1)
        return 1.0 + torch.pow(2.0, 1.0 - reg)

    def advance(self):
        return [self.step()]

    def _all_max(self, v: float) -> float:
        t = torch.tensor([v], dtype=torch.float64, device=self.x.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def step(self):
        s = self.solver
        self._maybe_rebalance(self.step_index)
        self._exchange()  # migration of the last step's leavers + fresh ghosts
        failure, st = None, None
        try:
            st = s.step()
        except (NumericalError, RuntimeError) as exc:  # raised on every rank below
            failure = exc
        n_own = self.n_own
        # one all-reduce: [any rank failed, owned active count, owned rho sum]
        v = torch.zeros(3, dtype=torch.float64, device=self.device)
        v[0] = 1.0 if failure is not None else 0.0
        if failure is None:
            v[1] = s.compute[:n_own].sum()
            v[2] = s.rho[:n_own].double().sum()
        v = v.to(self.x.device)
        dist.all_reduce(v)
        fail, n_act, rho_sum = v.tolist()
        if fail:
            raise failure if failure is not None else NumericalError(
                "another x-slab rank failed in this step")
        st.n_compute = int(n_act)  # all ranks' owned particles
        st.frac_compute = st.n_compute / max(1, self.n_global)
        if s.track_rho_variance:  # population variance over every rank's owned rows
            mean = rho_sum / max(1, self.n_global)
            d = torch.zeros(1, dtype=torch.float64, device=self.device)
            d[0] = ((s.rho[:n_own].double() - mean) ** 2).sum()
            d = d.to(self.x.device)
            dist.all_reduce(d)
            st.rho_var = float(d.item()) / max(1, self.n_global)
        s._resize_fluid(n_own)  # drop the ghost rows
        self.sim_time += st.dt
        self.step_index += 1
        return st


class DistributedPcisph(_ResidentRank):
    """RTS-PCISPH over x-slabs: at every major step migration and a fresh
    6-column ghost band (fast-region expansion reaches 4 blocks, smoothing 1
    more) on resident rows (``_ResidentRank``); the major step's correction
    loops then exchange the 2 inner ghost columns and fold the convergence
    scalars every iteration (``PcisphExchange``)."""

    def __init__(self, scene: Scene, device=None, halo: int = 6, inner: int = 2, jitter=None,
                 comm_device=None, velocity=None, balance: bool = True, rebalance_every: int = 0,
                 **kw):
        from .pcisph import PcisphSolver
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.part = SlabPartition.for_scene(scene, "pcisph", self.world, halo, balance)
        self.rebalance_every = rebalance_every
        self.inner = inner
        gid, fluid, wall, wsel = initial_ownership(scene, self.part, self.rank)
        self._keep_walls(wall)
        if jitter is not None:
            fluid = (fluid + jitter).astype(np.float32).astype(np.float64)
        if comm_device is None and dist.get_backend() == "gloo":
            comm_device = "cpu"
        self.driver = SlabDriver(self.part, self.rank, self.device, comm_device=comm_device)
        self.x = self.driver.x
        self.n_global = len(fluid)
        s = self.solver = PcisphSolver(scene, mode="rts", device=self.device, use_graphs=False,
                                       **kw)
        s._set_local_particles(None, wall[wsel], init=True)
        s.params.n_global = self.n_global
        fl = torch.as_tensor(fluid[gid].astype(np.float32), device=self.device)
        st = s._fresh_state(fl)
        st["xstar"] = fl.clone()
        if velocity is not None:  # (n_global, 3) initial velocities by global id
            st["vel"] = torch.as_tensor(np.asarray(velocity)[gid], device=self.device,
                                        dtype=st["vel"].dtype)
        self._init_rows(gid, st, halo)
        self.sim_time = 0.0
        self.step_index = 0
        self._majors = 0

    def _work_weights(self, n: int) -> torch.Tensor:
        """Refreshes per major of each owned row: region n is refreshed every
        VALIDITY_PERIOD[n] minor steps (pcisph.py:63-66), plus the per-row
        passes every particle takes."""
        from .pcisph import VALIDITY_PERIOD
        per = torch.as_tensor(VALIDITY_PERIOD, dtype=torch.float64, device=self.device)
        reg = self.solver.arena["region"][:n].long().clamp(1, len(VALIDITY_PERIOD) - 1)
        return 1.0 + self.solver.scene.minor_steps / per[reg]

    def _lists(self):
        s = self.solver
        bx = self.part.block_x(s.arena["pos"][:s.n_fluid, 0])
        owned = torch.zeros(s.n_fluid, dtype=torch.bool, device=self.device)
        owned[:self.n_own] = True
        lo, hi = self.driver.lo, self.driver.hi
        send, recv = {}, {}
        for q in self.x.neighbours():
            if q < self.rank:
                sm = owned & (bx < lo + self.inner)
                rm = (~owned) & (bx >= lo - self.inner) & (bx < lo)
            else:
                sm = owned & (bx >= hi - self.inner)
                rm = (~owned) & (bx >= hi) & (bx < hi + self.inner)
            # both sides list the rows in global-id order: a rank's local row
            # order is free (hole filling, arrivals, ghosts in message order)
            send[q] = self._by_gid(torch.nonzero(sm).reshape(-1))
            recv[q] = self._by_gid(torch.nonzero(rm).reshape(-1))
        return send, recv

    def _by_gid(self, idx: torch.Tensor) -> torch.Tensor:
        return idx[torch.argsort(self.solver.arena["sort_key"][idx])]

    def advance(self):
        s = self.solver
        self._maybe_rebalance(self._majors)
        self._majors += 1
        self._exchange()
        s.params.n_global = self.n_global
        send, recv = self._lists()
        s._xch = PcisphExchange(self.driver, send, recv)
        failure, rows = None, []
        try:
            rows = s.major_step()
        except (NumericalError, RuntimeError) as exc:  # raised on every rank below
            failure = exc
        finally:
            s._xch = None
        # one all-reduce: [any rank failed, refresh counts per minor step]
        from ._native import MAX_MINOR
        v = torch.zeros(1 + MAX_MINOR, dtype=torch.float64)
        v[0] = 1.0 if failure is not None else 0.0
        for j, r in enumerate(rows[:MAX_MINOR]):
            v[1 + j] = r.n_compute
        v = v.to(self.x.device)
        dist.all_reduce(v)
        v = v.tolist()
        if v[0]:
            raise failure if failure is not None else NumericalError(
                "another x-slab rank failed in this major step")
        for j, r in enumerate(rows):
            r.n_compute = int(v[1 + j])
            r.frac_compute = r.n_compute / max(1, self.n_global)
        self.sim_time = s.sim_time
        self.step_index = s.step_index
        return rows

    def major_step(self):
        return self.advance()


def rank_solver(kind: str, scene: Scene, comm, *args, **kw):
    """``WcsphSolver(..., comm=group)`` / ``PcisphSolver(..., comm=group)``: this
    process is one x-slab rank (one GPU per process; ``device`` defaults to
    the current CUDA device).  ``comm`` must be the default process group."""
    if comm is not dist.group.WORLD and comm != dist.group.WORLD:
        raise ValueError("comm must be torch.distributed.group.WORLD (x-slab ranks use the "
                         "default process group)")
    kw.pop("use_graphs", None)  # ranks launch per kernel (the row count changes)
    names = ("mode",) + (("dt_cap", "pin_region", "apply_correction", "track_rho_variance",
                          "audit_neighbors", "n_regions") if kind == "wcsph" else
                         ("dt", "schedule", "pin_region", "audit_neighbors", "iteration_cap",
                          "local_attempts", "n_regions"))
    kw.update(zip(names, args))
    if kw.get("device") is None:
        kw["device"] = torch.device("cuda", torch.cuda.current_device())
    if kind == "wcsph":
        return DistributedWcsph(scene, **kw)
    if kw.pop("mode", "rts") != "rts":
        raise ValueError("x-slab ranks run RTS-PCISPH (mode='rts')")
    return DistributedPcisph(scene, **kw)
