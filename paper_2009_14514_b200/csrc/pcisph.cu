// RTS-PCISPH kernels (reference: /root/reference/pkg/src/rts_sph/pcisph.py).
//
// Neighbour tables are materialised (the minor steps deliberately reuse
// stale tables, pcisph.py:7-10, 553-557): `nbr` row i holds reference
// particle indices in the reference's fill order, `cnt[i]` its length.
// Predicted positions live in `xs` (32-byte rows, common.cuh XsRow: fluid
// rows fp64 x* and fp32 p; wall rows the static position and -1), so every
// pair kernel reads one 256-bit record per neighbour regardless of its kind.
//
// Per correction iteration the host enqueues
//   motion   x* for all fluid (first iteration / after a revert) or only for
//            the previous force set (x* depends on f_p alone, which changed
//            only there -- bit-identical to recomputing all, pcisph.py:202-213)
//   sets     turn | S_e | S_ob membership -> compact pred/force lists, S_ob
//            refresh from the observed-block mask (pcisph.py:637-643)
//   density  rho*, err over the pred list; Jacobi pressure update for force
//            members (pcisph.py:216-235, 432-437)
//   se       S_e = err > eta_max/2, S_e blocks, max err, sum rho* (fixed-order
//            two-level reduction: deterministic), any(S_e) (pcisph.py:662-684)
//   observed observed-block mask (regions.py:110-125)
//   pforces  pressure forces over the force list (pcisph.py:238-271)
#include "common.cuh"

// density pass variants (scripts/build_variant.sh A/B)
#ifndef RTS_DENS_PF
#define RTS_DENS_PF 1
#endif
#ifndef RTS_DENS_CH
#define RTS_DENS_CH 2
#endif
#ifndef RTS_DENS_MINB
#define RTS_DENS_MINB 8
#endif
#ifndef RTS_PFOR_PF
#define RTS_PFOR_PF 1
#endif
#ifndef RTS_LG_CH
#define RTS_LG_CH 3
#endif
#ifndef RTS_PFOR_CH
#define RTS_PFOR_CH 2
#endif
#ifndef RTS_RF_TWO_PHASE
#define RTS_RF_TWO_PHASE 1  // one-thread refresh: slots in the scan, ids + f_ext in a second loop
#endif
#ifndef RTS_RF_SBUF
#define RTS_RF_SBUF 32  // row entries per thread kept in shared memory by the two-phase refresh
#endif
#ifndef RTS_RF_P2
#define RTS_RF_P2 4  // phase-2 entries in flight per thread
#endif
#ifndef RTS_MOTION_1PT
#define RTS_MOTION_1PT 1  // all-particle motion: one particle per thread
#endif
#ifndef RTS_INTEG_1PT
#define RTS_INTEG_1PT 0  // integrator: one particle per thread (measured +25 us per launch: not kept)
#endif
#ifndef RTS_MAJOR_FORK
#define RTS_MAJOR_FORK 1  // major-step graph: gather || levels
#endif
#ifndef RTS_SETS_CAP
#define RTS_SETS_CAP (148 * 32)
#endif
#ifndef RTS_RLIST_CAP
#define RTS_RLIST_CAP (148 * 64)
#endif
#ifndef RTS_INTEG_GRID4
#define RTS_INTEG_GRID4 1
#endif
#ifndef RTS_PFOR_MINB
#define RTS_PFOR_MINB 7
#endif
#ifndef RTS_PAIR_CARVEOUT
#define RTS_PAIR_CARVEOUT 0  // shared-memory carveout (%) asked for the pair passes (0: largest L1; -1: driver default)
#endif
#ifndef RTS_PAIR_CAP
#define RTS_PAIR_CAP (148 * 32)  // grid cap of the pair passes (CTAs of kThreads)
#endif

using namespace rts;

namespace {

constexpr int kThreads = 128;
constexpr int kRedBlocks = 592;  // fixed partial count -> deterministic sums

__constant__ int kValidity[5] = {0, 1, 2, 4, 4};  // pcisph.py:66

// S_ob membership of a block: static transition bit (block_tmp) or next to
// an S_e block of generation `gen` without being one (regions.py:119-125)
RTS_DEV bool observed_block(const RtsBuffers &b, int c, int gen) {
    return b.block_tmp[c] || (b.near_stamp[c] == gen && b.se_stamp[c] != gen);
}

// ghost rows (x-slab ranks) are neighbours only: never refreshed, predicted,
// corrected or integrated here -- their owner computes them
RTS_DEV bool is_ghost(const RtsBuffers &b, int i) { return b.ghost && b.ghost[i]; }

// loop control flags (ctl may be null for callers outside a solver)
RTS_DEV bool loop_done(const RtsBuffers &b) { return b.ctl && b.ctl->done; }
RTS_DEV bool major_stopped(const RtsBuffers &b) { return b.ctl && b.ctl->stop_major; }
// iteration kernels skip when the loop has finished or a fatal flag is set
#define RTS_ITER_GUARD() if (fatal(b.ctr) || loop_done(b)) return
#define RTS_MINOR_GUARD() if (fatal(b.ctr) || major_stopped(b)) return

RTS_DEV int trunc_axis(double x, double o, double inv, int n) {
    // int((x - o) * inv) then clamp (grid.py:116-131)
    const double v = xmul(xsub(x, o), inv);
    if (!(v >= 0.0)) return 0;
    if (v >= (double)(n - 1)) return n - 1;
    return (int)v;
}

RTS_DEV XsRow *xs_rows(const RtsBuffers &b) { return reinterpret_cast<XsRow *>(b.xs); }

// wall rows of xs (static positions, marker -1)
__global__ void k_xs_walls(const __grid_constant__ RtsParams p, RtsBuffers b) {
    const int nb = p.n_bound;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nb; t += gridDim.x * blockDim.x) {
        const int j = p.n_fluid + t;
        st_xs(xs_rows(b) + j, b.pos[3 * j], b.pos[3 * j + 1], b.pos[3 * j + 2], -1.0);
    }
}

// candidate copies of the major grid: cpos[k] = (pos[order[k]], bits of
// order[k]), slot_of
__global__ void k_gather(const __grid_constant__ RtsParams p, RtsBuffers b) {
    if (fatal(b.ctr)) return;
    const int n = b.ctr->n_sorted;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int j = rts_safe_idx(b.ctr, b.order[k], p.n_fluid + p.n_bound, 301, 0);
        const float x = b.pos[3 * j], y = b.pos[3 * j + 1], z = b.pos[3 * j + 2];
        reinterpret_cast<float4 *>(b.cpos)[k] = make_float4(x, y, z, __int_as_float(j));
        if (b.cx) b.cx[k] = x, b.cy[k] = y, b.cz[k] = z;
        if (j < p.n_fluid) b.slot_of[j] = k;
    }
    if (b.cx && blockIdx.x == 0 && threadIdx.x == 0) b.ctr->soa_fresh = 1;
}

// _assign_major_regions per-particle tail (pcisph.py:531-534)
__global__ void k_major_particles(const __grid_constant__ RtsParams p, RtsBuffers b) {
    if (fatal(b.ctr)) return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.n_fluid;
         i += gridDim.x * blockDim.x) {
        const int8_t r = b.block_field[b.fluid_cells[i]];
        b.region[i] = r;
        b.validity[i] = kValidity[r < 0 ? 0 : (r > 4 ? 4 : r)];
        b.compute[i] = 1;
        b.in_se[i] = 0;
    }
}

// refresh list: particles whose tables are renewed this minor step
// The refresh list is built in CSR (block-key) order, not particle order:
// consecutive lanes then belong to the same or z-adjacent blocks, so their
// candidate spans coincide and a warp's span loads collapse onto a few cache
// lines instead of one line per lane (-16 % on the full refresh).  The
// table-driven kernels keep particle order, where consecutive lanes read
// consecutive rows.
__global__ void __launch_bounds__(256) k_refresh_list(const __grid_constant__ RtsParams p,
                                                      RtsBuffers b, int all) {
    RTS_MINOR_GUARD();
    const int nf = p.n_fluid;
    const int ns = b.ctr->n_sorted;
    const int stride = gridDim.x * blockDim.x;
    for (int base = blockIdx.x * blockDim.x; base < ns; base += stride) {
        const int k = base + threadIdx.x;
        const int i = k < ns ? b.order[k] : nf;
        const bool r = i < nf && (all || b.compute[i]) && !is_ghost(b, i);
        block_append2<256>(r, i, b.active, &b.ctr->n_compute, false, 0, nullptr, nullptr);
    }
}

// ---- search_into on the (stale) major grid (grid.py:88-152) fused with the
// external forces of the refreshed particle (pcisph.py:174-199) ------------
//
// Membership: candidates are classified in fp32 with a +-1e-5 relative band
// around h^2; only candidates inside the band take the exact fp64 test, so
// membership equals the reference's fp64 `r2 < h2` exactly.  Table rows are
// filled in the reference's order (blocks in (ax, ay, az) order, CSR order
// inside a block).  The viscosity sum of f_ext is a fixed-order tree
// (deterministic; f_ext parity bar 1e-4).
struct RefreshConsts {
    float h2_lo, h2_hi;
    float hf, visc_f;  // h and mu m^2 c_visc / rho0^2 for the fp32 viscosity terms
};

RTS_DEV RefreshConsts refresh_consts(const RtsParams &p) {
    RefreshConsts k;
    k.h2_lo = (float)(p.h2 * (1.0 - 1e-5));
    k.h2_hi = (float)(p.h2 * (1.0 + 1e-5));
    k.hf = (float)p.h;
    // mu m^2 c_visc / rho0^2 (pcisph.py:183-196)
    k.visc_f = (float)xmul(xmul(xmul(p.mu, xmul(p.mass, p.mass)), p.c_visc),
                           xdiv(1.0, xmul(p.rho0, p.rho0)));
    return k;
}

RTS_DEV bool is_neighbour(const RefreshConsts &k, const RtsParams &p, float fxi, float fyi,
                          float fzi, float4 o) {
    const float ex = __fsub_rn(fxi, o.x), ey = __fsub_rn(fyi, o.y), ez = __fsub_rn(fzi, o.z);
    const float r2f = __fmaf_rn(ex, ex, __fmaf_rn(ey, ey, __fmul_rn(ez, ez)));
    if (r2f > k.h2_hi) return false;
    if (r2f < k.h2_lo) return true;
    return exact_neighbour(p.h2, fxi, fyi, fzi, o.x, o.y, o.z);
}

// viscosity term of one table entry j for particle i (pcisph.py:183-196), in
// fp32 like the thread path of refresh_one, accumulated in fp64
RTS_DEV void visc_term(const RefreshConsts &k, const RtsParams &p, const RtsBuffers &b, int i,
                       int j, double xi, double yi, double zi, float4 pj, double vxi, double vyi,
                       double vzi, double &fx, double &fy, double &fz) {
    if (j >= p.n_fluid || j == i) return;
    const float dx = (float)xi - pj.x, dy = (float)yi - pj.y, dz = (float)zi - pj.z;
    const float r = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
    if (r >= k.hf) return;
    const float lap = k.visc_f * (k.hf - r);
    fx += (double)(lap * (b.vel[3 * j] - (float)vxi));
    fy += (double)(lap * (b.vel[3 * j + 1] - (float)vyi));
    fz += (double)(lap * (b.vel[3 * j + 2] - (float)vzi));
}

RTS_DEV void finish_search(const RtsParams &p, const RtsBuffers &b, int i, int cntn) {
    if (cntn > p.width) {
        atomicOr(&b.ctr->err_flags, RTS_ERR_OVERFLOW);
        atomicAdd((unsigned long long *)&b.ctr->overflow, (unsigned long long)(cntn - p.width));
        cntn = p.width;
    }
    b.cnt[i] = cntn;
}

RTS_DEV void finish_refresh(const RtsParams &p, const RtsBuffers &b, int i, int cntn, double fx,
                            double fy, double fz) {
    if (cntn > p.width) {
        atomicOr(&b.ctr->err_flags, RTS_ERR_OVERFLOW);
        atomicAdd((unsigned long long *)&b.ctr->overflow, (unsigned long long)(cntn - p.width));
        cntn = p.width;
    }
    b.cnt[i] = cntn;
    b.force[3 * i] = (float)xadd(fx, xmul(p.mass, p.gravity[0]));
    b.force[3 * i + 1] = (float)xadd(fy, xmul(p.mass, p.gravity[1]));
    b.force[3 * i + 2] = (float)xadd(fz, xmul(p.mass, p.gravity[2]));
}

// One CSR span [k0, k1) of the one-thread-per-particle refresh (G = 1):
// candidates classified 32 at a time, members emitted in candidate order
// (with EXT, their viscosity terms summed as they are emitted).
template <bool EXT>
RTS_DEV void refresh_span(const RtsParams &p, const RtsBuffers &b, const RefreshConsts &k, int i,
                          int k0, int k1, float fxi, float fyi, float fzi, double vxi, double vyi,
                          double vzi, int *row, size_t S, int &cntn, double &vfx, double &vfy,
                          double &vfz, int *sbuf) {
    const float4 *cpos = reinterpret_cast<const float4 *>(b.cpos);
    // Branch-free classification of 32 candidates at a time: two
    // 32-bit masks (r2 < h2_lo: member; r2 > h2_hi: not) built
    // from the sign bits of r2 - bound with one funnel shift per
    // candidate; the rare in-band candidates then take the exact
    // fp64 test, and the members are emitted in candidate order.
    // Reads run up to 3 slots past the span (cpos is padded).
    const bool soa = RTS_SOA && b.cx != nullptr && b.ctr->soa_fresh;
    for (int cb = soa ? (k0 & ~3) : k0; cb < k1; cb += 32) {
        const int n = min(32, k1 - cb);
        const float4 *cp = cpos + cb;
        unsigned mem = 0u, out = 0u;  // first candidate ends in the top bit
        if (soa) {  // x / y / z copies: 4 candidates per load, fp32x2 tests
            unsigned amb;
            classify_soa(b.cx, b.cy, b.cz, cb, n, k0, fxi, fyi, fzi, k.h2_lo, k.h2_hi, mem,
                         amb);
            while (amb) {
                const int q = __ffs(amb) - 1;
                amb &= amb - 1u;
                const float4 o = cp[q];
                if (exact_neighbour(p.h2, fxi, fyi, fzi, o.x, o.y, o.z)) mem |= 1u << q;
            }
        } else {
            for (int u = 0; u < n; u += 4) {
                float4 ob[4];
#pragma unroll
                for (int v = 0; v < 4; ++v) ob[v] = cp[u + v];
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const float ex = __fsub_rn(fxi, ob[v].x), ey = __fsub_rn(fyi, ob[v].y),
                                ez = __fsub_rn(fzi, ob[v].z);
                    const float r2f = __fmaf_rn(ex, ex, __fmaf_rn(ey, ey, __fmul_rn(ez, ez)));
                    mem = __funnelshift_l(__float_as_uint(__fsub_rn(r2f, k.h2_lo)), mem, 1);
                    out = __funnelshift_l(__float_as_uint(__fsub_rn(k.h2_hi, r2f)), out, 1);
                }
            }
            const int nr = (n + 3) & ~3;  // candidates classified
            // bit (nr-1-u) <-> candidate u; reverse so bit u <-> candidate u
            const unsigned valid = n == 32 ? 0xffffffffu : ((1u << n) - 1u);
            mem = (__brev(mem) >> (32 - nr)) & valid;
            out = (__brev(out) >> (32 - nr)) & valid;
            {
                unsigned amb = valid & ~mem & ~out;
                while (amb) {
                    const int q = __ffs(amb) - 1;
                    amb &= amb - 1u;
                    const float4 o = cp[q];
                    if (exact_neighbour(p.h2, fxi, fyi, fzi, o.x, o.y, o.z)) mem |= 1u << q;
                }
            }
        }
        if (!EXT) {
            while (mem) {
                const int q = __ffs(mem) - 1;
                mem &= mem - 1u;
                if (cntn < p.width) __stcs(row + cntn * S, __float_as_int(cp[q].w));
                ++cntn;
            }
            continue;
        }
        if (RTS_RF_TWO_PHASE) {
            // phase 1: the members' CSR slots, in candidate (= row) order;
            // refresh_one's phase 2 turns them into ids and sums f_ext
            while (mem) {
                const int q = __ffs(mem) - 1;
                mem &= mem - 1u;
                if (cntn < RTS_RF_SBUF) sbuf[cntn * kThreads] = cb + q;
                else if (cntn < p.width) row[cntn * S] = cb + q;
                ++cntn;
            }
            continue;
        }
        // members in candidate (= row) order, four at a time: the
        // candidate copy (L1-hot) gives j and pos_j, so the row is
        // written and its viscosity term (fp32, fp64 row-order sum;
        // pcisph.py:183-196) taken without re-reading the row
        while (mem) {
            float4 o[4];
            float vj[4][3];
            int nq = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                o[u] = make_float4(fxi, fyi, fzi, __int_as_float(i));
                if (mem) {
                    o[u] = cp[__ffs(mem) - 1];
                    mem &= mem - 1u;
                    nq = u + 1;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int j = __float_as_int(o[u].w);
                const int jc = j < p.n_fluid ? j : i;
                vj[u][0] = b.vel[3 * jc];
                vj[u][1] = b.vel[3 * jc + 1];
                vj[u][2] = b.vel[3 * jc + 2];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (u >= nq) break;
                const int j = __float_as_int(o[u].w);
                if (cntn < p.width) {
                    __stcs(row + cntn * S, j);
                    if (j < p.n_fluid && j != i) {
                        const float dx = fxi - o[u].x, dy = fyi - o[u].y,
                                    dz = fzi - o[u].z;
                        const float r = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                        if (r < k.hf) {
                            const float lap = k.visc_f * (k.hf - r);
                            vfx += (double)(lap * (vj[u][0] - (float)vxi));
                            vfy += (double)(lap * (vj[u][1] - (float)vyi));
                            vfz += (double)(lap * (vj[u][2] - (float)vzi));
                        }
                    }
                }
                ++cntn;
            }
        }
    }
}

// One thread (G = 1) or one G-lane group per refreshed particle, chosen from
// the list length against the grid (pass_blocks): on large scenes the full
// refresh at a major-step start keeps one thread per particle (adjacent lanes
// share candidate spans -> few L1 lines per load) and, with G = 1 and EXT,
// forms the viscosity sum while it emits the row (ids and positions come
// from the candidate copy, so the row is never re-read); the short later
// lists (regions 1-2) and every list of a small scene use 8- or 32-lane
// groups so the launch still has enough independent loads in flight
// (region-1 particles scan 125 blocks, ~1300 candidates).
// EXT = false: the bare search (BlockGrid.search_into, grid.py:297-331) --
// rows and counts only, `lay_in` block layers for this particle.
//
// Culling (D >= 0): a block of the stale window is scanned only if one of
// its candidates can lie within h of the particle -- candidates sit in the
// block of their position at the rebuild and have moved by at most D per
// coordinate since (the integrator's bound, RtsCounters.disp_*).  Whole
// block columns farther than h in x-y are skipped and each column's span is
// clipped to the z blocks within +-sqrt(h^2 - d_xy^2) (+ D).  Rows are
// unchanged: skipped blocks hold no member, and the kept blocks stay
// contiguous slot ranges in the reference's order.  The region-1 two-layer
// windows of the later minor steps (125 blocks) shrink ~5x.
template <int G, bool EXT = true>
RTS_DEV void refresh_one(const RtsParams &p, const RtsBuffers &b, const RefreshConsts &k, int i,
                         int two_layer_r1, int lane, unsigned gmask, int gshift, int lay_in = 0,
                         double D = -1.0, int *sbuf = nullptr) {
    const float4 *cpos = reinterpret_cast<const float4 *>(b.cpos);
    const int nx = p.dims[0], ny = p.dims[1], nz = p.dims[2];
    RTS_CHECK_IDX(b.ctr, i, p.n_fluid, 302);
    const float fxi = b.pos[3 * i], fyi = b.pos[3 * i + 1], fzi = b.pos[3 * i + 2];
    const double xi = fxi, yi = fyi, zi = fzi;
    const int lay = lay_in > 0 ? lay_in : ((two_layer_r1 && b.region[i] == 1) ? 2 : 1);
    const int cx = trunc_axis(xi, p.origin[0], p.inv_block, nx);
    const int cy = trunc_axis(yi, p.origin[1], p.inv_block, ny);
    const int cz = trunc_axis(zi, p.origin[2], p.inv_block, nz);
    const int z0 = max(0, cz - lay), z1 = min(nz - 1, cz + lay);
    const unsigned lt = (1u << lane) - 1u;
    int cntn = 0;
    // G == 1 && EXT: the viscosity sum is formed while the row is emitted
    const double vxi = EXT ? b.vel[3 * i] : 0.0, vyi = EXT ? b.vel[3 * i + 1] : 0.0,
                 vzi = EXT ? b.vel[3 * i + 2] : 0.0;
    double vfx = 0.0, vfy = 0.0, vfz = 0.0;
    int *row = b.nbr + i;  // entry q at row[q * S]
    const size_t S = p.nbr_stride;
    const bool cull = D >= 0.0;
    // the block ranges of the (2L+1)^3 window that can hold a candidate within
    // h: +-(h + D) around the particle, per axis (computed once per particle)
    int ax0 = max(0, cx - lay), ax1 = min(nx - 1, cx + lay);
    int ay0 = max(0, cy - lay), ay1 = min(ny - 1, cy + lay);
    int za = z0, zb = z1;
    double hw2 = 0.0;
    if (cull) {
        const double w = p.h * (1.0 + 1e-6) + D + 1e-9 * p.block_size;
        hw2 = p.h2 * (1.0 + 2e-6);
        auto lo = [&](double x, double o) { return floor((x - w - o) * p.inv_block); };
        auto hi = [&](double x, double o) { return floor((x + w - o) * p.inv_block); };
        ax0 = max(ax0, (int)fmax(lo(xi, p.origin[0]), -1.0));
        ax1 = min(ax1, (int)fmin(hi(xi, p.origin[0]), (double)nx));
        ay0 = max(ay0, (int)fmax(lo(yi, p.origin[1]), -1.0));
        ay1 = min(ay1, (int)fmin(hi(yi, p.origin[1]), (double)ny));
        za = max(za, (int)fmax(lo(zi, p.origin[2]), -1.0));
        zb = min(zb, (int)fmin(hi(zi, p.origin[2]), (double)nz));
    }
    const double B = p.block_size;
    for (int ax = ax0; ax <= ax1; ++ax) {
        double ddx = 0.0;
        if (cull) {  // x distance from the column's candidates (stale extent +- D)
            const double xl = ax == 0 ? -1e300 : p.origin[0] + ax * B - D;
            const double xh = ax == nx - 1 ? 1e300 : p.origin[0] + (ax + 1) * B + D;
            ddx = xi < xl ? xl - xi : (xi > xh ? xi - xh : 0.0);
        }
        for (int ay = ay0; ay <= ay1; ++ay) {
            const int base = (ax * ny + ay) * nz;
            if (cull) {  // corner columns: x-y distance
                const double yl = ay == 0 ? -1e300 : p.origin[1] + ay * B - D;
                const double yh = ay == ny - 1 ? 1e300 : p.origin[1] + (ay + 1) * B + D;
                const double ddy = yi < yl ? yl - yi : (yi > yh ? yi - yh : 0.0);
                if (ddx * ddx + ddy * ddy >= hw2) continue;  // no candidate within h
            }
            if (za > zb) continue;
            RTS_CHECK(b.ctr, base + zb + 1 <= p.n_cells, 303);
            const int k0 = b.starts[base + za], k1 = b.starts[base + zb + 1];
            RTS_CHECK(b.ctr, 0 <= k0 && k0 <= k1 && k1 <= b.ctr->n_sorted, 304);
            if (G == 1) {
                refresh_span<EXT>(p, b, k, i, k0, k1, fxi, fyi, fzi, vxi, vyi, vzi, row, S, cntn,
                                  vfx, vfy, vfz, sbuf);
            } else {
                for (int kb = k0; kb < k1; kb += G) {
                    const int kk = kb + lane;
                    const float4 o = kk < k1 ? cpos[kk] : make_float4(0.f, 0.f, 0.f, 0.f);
                    const bool in = kk < k1 && is_neighbour(k, p, fxi, fyi, fzi, o);
                    const unsigned m =
                        (__ballot_sync(gmask, in) >> gshift) & (G == 32 ? 0xffffffffu : ((1u << G) - 1u));
                    if (in) {
                        const int slot = cntn + __popc(m & lt);
                        if (slot < p.width) __stcs(row + slot * S, __float_as_int(o.w));
                    }
                    cntn += __popc(m);
                }
            }
        }
    }
    if (G > 1) __syncwarp(gmask);
    if (!EXT) {
        if (lane == 0) finish_search(p, b, i, cntn);
        return;
    }
    const int nrow = min(cntn, p.width);
    if (G == 1 && RTS_RF_TWO_PHASE) {
        // phase 2, uniform across the warp (every lane walks its own row,
        // ~30 entries): slot -> candidate copy (id, current position) ->
        // velocity; the row entry becomes the id and the viscosity term is
        // summed in row order (fp32 terms, fp64 sum; pcisph.py:183-196).
        // The per-chunk emission this replaces ran at ~13 of 32 lanes.
        const int nsorted = b.ctr->n_sorted;
        for (int q0 = 0; q0 < nrow; q0 += RTS_RF_P2) {
            int sl[RTS_RF_P2];
            float4 o[RTS_RF_P2];
            float vj[RTS_RF_P2][3];
#pragma unroll
            for (int u = 0; u < RTS_RF_P2; ++u)
                sl[u] = q0 + u < nrow
                            ? rts_safe_idx(b.ctr,
                                           q0 + u < RTS_RF_SBUF ? sbuf[(q0 + u) * kThreads]
                                                                : row[(q0 + u) * S],
                                           nsorted, 305, 0)
                            : -1;
#pragma unroll
            for (int u = 0; u < RTS_RF_P2; ++u)
                o[u] = sl[u] >= 0 ? cpos[sl[u]] : make_float4(fxi, fyi, fzi, __int_as_float(i));
#pragma unroll
            for (int u = 0; u < RTS_RF_P2; ++u) {
                const int j = __float_as_int(o[u].w);
                const int jc = j < p.n_fluid ? j : i;
                vj[u][0] = b.vel[3 * jc];
                vj[u][1] = b.vel[3 * jc + 1];
                vj[u][2] = b.vel[3 * jc + 2];
            }
#pragma unroll
            for (int u = 0; u < RTS_RF_P2; ++u) {
                if (q0 + u >= nrow) break;
                const int j = __float_as_int(o[u].w);
                __stcs(row + (q0 + u) * S, j);
                if (j < p.n_fluid && j != i) {
                    const float dx = fxi - o[u].x, dy = fyi - o[u].y, dz = fzi - o[u].z;
                    const float r = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                    if (r < k.hf) {
                        const float lap = k.visc_f * (k.hf - r);
                        vfx += (double)(lap * (vj[u][0] - (float)vxi));
                        vfy += (double)(lap * (vj[u][1] - (float)vyi));
                        vfz += (double)(lap * (vj[u][2] - (float)vzi));
                    }
                }
            }
        }
    }
    double fx = vfx, fy = vfy, fz = vfz;
    if (G > 1) {  // (G == 1: summed above, while the row was emitted)
        for (int q = lane; q < nrow; q += G) {
            const int j = row[q * S];
            const float4 pj = make_float4(b.pos[3 * j], b.pos[3 * j + 1], b.pos[3 * j + 2], 0.f);
            visc_term(k, p, b, i, j, xi, yi, zi, pj, vxi, vyi, vzi, fx, fy, fz);
        }
    }
    if (G > 1) {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            fx = xadd(fx, __shfl_xor_sync(gmask, fx, o, G));
            fy = xadd(fy, __shfl_xor_sync(gmask, fy, o, G));
            fz = xadd(fz, __shfl_xor_sync(gmask, fz, o, G));
        }
    }
    if (lane == 0) finish_refresh(p, b, i, cntn, fx, fy, fz);
}

#ifndef RTS_REF_MID
#define RTS_REF_MID 8  // lanes per particle for mid-size refresh lists (8, 4 or 1)
#endif
#ifndef RTS_CULL_G1
#define RTS_CULL_G1 0  // culling in the one-thread-per-particle path (lanes diverge)
#endif
#ifndef RTS_REF_MINB
#define RTS_REF_MINB 6  // 70 registers: 331 us full refresh vs 342 at 8 CTAs/SM (64 regs), 355 at 5
#endif

__global__ void __launch_bounds__(kThreads, RTS_REF_MINB) k_refresh(const __grid_constant__ RtsParams p,
                                                      RtsBuffers b, int two_layer_r1) {
    // phase-1 member slots of the one-thread path: the first RTS_RF_SBUF
    // entries of each row stay on chip (entry q of thread t at [q][t]:
    // conflict-free), the rest go through the row itself
    __shared__ int s_slots[(RTS_RF_SBUF > 0 ? RTS_RF_SBUF : 1) * kThreads];
    RTS_MINOR_GUARD();
    const int n = b.ctr->n_compute;
    const RefreshConsts k = refresh_consts(p);
    const int nthreads = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int wl = threadIdx.x & 31;
    // displacement bound of the candidates since the rebuild (+1e-5 relative:
    // measured in fp32); x-slab ranks: ghosts move on other ranks -> no culling
    const double D = b.ghost ? -1.0
                             : 1.00001 * ((double)b.ctr->disp_total + (double)b.ctr->disp_cur);
    if ((long long)n * 32 <= nthreads) {
        for (int t = tid / 32; t < n; t += nthreads / 32)
            refresh_one<32>(p, b, k, b.active[t], two_layer_r1, wl, 0xffffffffu, 0, 0, D);
    } else if ((long long)n * 8 <= nthreads && RTS_REF_MID == 8) {
        const int lane = wl & 7, gshift = wl & ~7;
        const unsigned gmask = 0xffu << gshift;
        for (int t = tid / 8; t < n; t += nthreads / 8)
            refresh_one<8>(p, b, k, b.active[t], two_layer_r1, lane, gmask, gshift, 0, D);
    } else if ((long long)n * 4 <= nthreads && RTS_REF_MID == 4) {
        const int lane = wl & 3, gshift = wl & ~3;
        const unsigned gmask = 0xfu << gshift;
        for (int t = tid / 4; t < n; t += nthreads / 4)
            refresh_one<4>(p, b, k, b.active[t], two_layer_r1, lane, gmask, gshift, 0, D);
    } else {
        for (int t = tid; t < n; t += nthreads)
            refresh_one<1>(p, b, k, b.active[t], two_layer_r1, 0, 0u, 0, 0, RTS_CULL_G1 ? D : -1.0,
                           s_slots + threadIdx.x);
    }
}

// BlockGrid.search_into: rows for the refresh list in `active`, layers[t]
// block layers for entry t (grid.py:88-152)
__global__ void __launch_bounds__(kThreads) k_search(const __grid_constant__ RtsParams p,
                                                     RtsBuffers b, const int8_t *layers, int n) {
    const RefreshConsts k = refresh_consts(p);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        refresh_one<1, false>(p, b, k, b.active[t], 0, 0, 0u, 0, layers[t]);
}

// x* = pos + dt * (vel + dt/m (f_ext + f_p)) (pcisph.py:202-213), kept in
// fp64 in the xs row (the row's p is the density pass's)
RTS_DEV void motion_one(const RtsParams &p, const RtsBuffers &b, int i, double dt_inv_m) {
    double xs[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double f = xadd((double)b.force[3 * i + a], (double)b.f_p[3 * i + a]);
        const double v = xadd((double)b.vel[3 * i + a], xmul(dt_inv_m, f));
        xs[a] = xadd((double)b.pos[3 * i + a], xmul(p.dt, v));
    }
    // the whole 32-byte row (a partial-sector store costs a read-modify-write
    // in DRAM once the rows outgrow L2, cfg4/cfg5): p is re-stored unchanged
    XsRow *r = xs_rows(b) + i;
    st_xs(r, xs[0], xs[1], xs[2], r->p);
}

// the fp64 p of row i (and its fp32 public mirror)
RTS_DEV void set_p(const RtsBuffers &b, int i, double pr) {
    b.pres[i] = (float)pr;
    b.xs[4 * i + 3] = pr;
}

// restore p, f_p of particle i from the local-phase entry snapshot
RTS_DEV void restore_one(const RtsBuffers &b, int i) {
    set_p(b, i, b.snap_p[i]);
    b.f_p[3 * i] = b.snap_fp[3 * i];
    b.f_p[3 * i + 1] = b.snap_fp[3 * i + 1];
    b.f_p[3 * i + 2] = b.snap_fp[3 * i + 2];
}

// all = 1: every fluid particle; 0: the previous force list; -1: ctl->motion_all.
// The all-particle pass streams four particles per thread with float4 loads.
// A revert decided by the previous iteration's control (ctl->snap_op == 2,
// which also sets motion_all) restores p, f_p here, before x* is formed.
__global__ void k_motion(const __grid_constant__ RtsParams p, RtsBuffers b, int all) {
    RTS_ITER_GUARD();
    const bool restore = b.ctl && b.ctl->snap_op == 2;
    // first iteration of a minor step: p = 0, f_p = 0 for all fluid
    // (pcisph.py:570-571) folded in here; the refresh phase ends now
    const bool zero = b.ctl && b.ctl->it == 0;
    if (zero && blockIdx.x == 0 && threadIdx.x == 0)
        b.ctl->stats[b.ctl->minor].t_refreshed = gtimer();
    if (all < 0) all = b.ctl->motion_all;
    if (restore || zero) all = 1;
    const double dim = xmul(p.dt, p.inv_mass);
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    if (!all) {
        const int n = b.ctl->prev_force;
        for (int t = tid; t < n; t += nt) {
            const int i = rts_safe_idx(b.ctr, b.list3[t], p.n_fluid, 501, 0);
            if (!is_ghost(b, i)) motion_one(p, b, i, dim);
        }
        return;
    }
    const int nf = p.n_fluid, ng = nf / 4;
    XsRow *xsr = xs_rows(b);
    if (RTS_MOTION_1PT) {
        // one particle per thread: every thread of the grid streams (the
        // four-per-thread path below left 3/4 of them idle), a warp's loads
        // and its 32-byte row stores each cover one contiguous range
        for (int i = tid; i < nf; i += nt) {
            float fe[3], fp[3], v[3], x[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                fe[a] = b.force[3 * i + a];
                v[a] = b.vel[3 * i + a];
                x[a] = b.pos[3 * i + a];
            }
            double pr;
            if (restore) {
                pr = b.snap_p[i];
#pragma unroll
                for (int a = 0; a < 3; ++a) fp[a] = b.snap_fp[3 * i + a];
            } else if (zero) {
                pr = 0.0;
                fp[0] = fp[1] = fp[2] = 0.f;
            } else {
                pr = xsr[i].p;
#pragma unroll
                for (int a = 0; a < 3; ++a) fp[a] = b.f_p[3 * i + a];
            }
            if (restore || zero) {
#pragma unroll
                for (int a = 0; a < 3; ++a) b.f_p[3 * i + a] = fp[a];
                b.pres[i] = (float)pr;
            }
            if (is_ghost(b, i)) continue;  // x* / p of ghost rows: the owner's (halo)
            double xs[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const double vv = xadd((double)v[a], xmul(dim, xadd((double)fe[a], (double)fp[a])));
                xs[a] = xadd((double)x[a], xmul(p.dt, vv));
            }
            st_xs(xsr + i, xs[0], xs[1], xs[2], pr);
        }
        return;
    }
    for (int g = tid; g < ng; g += nt) {
        float fe[12], fp[12], v[12], x[12];
        load12(b.force, g, fe);
        load12(b.vel, g, v);
        load12(b.pos, g, x);
        double pr[4] = {0.0, 0.0, 0.0, 0.0};
        if (zero) {
#pragma unroll
            for (int c = 0; c < 12; ++c) fp[c] = 0.f;
        } else {
            load12(restore ? b.snap_fp : b.f_p, g, fp);
            if (restore) {
                const double2 s01 = reinterpret_cast<const double2 *>(b.snap_p)[2 * g];
                const double2 s23 = reinterpret_cast<const double2 *>(b.snap_p)[2 * g + 1];
                pr[0] = s01.x, pr[1] = s01.y, pr[2] = s23.x, pr[3] = s23.y;
            }
        }
        if (restore || zero) {
            store12(b.f_p, g, fp);
            reinterpret_cast<float4 *>(b.pres)[g] =
                make_float4((float)pr[0], (float)pr[1], (float)pr[2], (float)pr[3]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double xs[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int c = 3 * q + a;
                const double vv = xadd((double)v[c], xmul(dim, xadd((double)fe[c], (double)fp[c])));
                xs[a] = xadd((double)x[c], xmul(p.dt, vv));
            }
            if (is_ghost(b, 4 * g + q)) continue;
            // whole 32-byte rows (see motion_one); p unchanged unless zeroed / restored
            st_xs(xsr + 4 * g + q, xs[0], xs[1], xs[2], (restore || zero) ? pr[q] : xsr[4 * g + q].p);
        }
    }
    for (int i = 4 * ng + tid; i < nf; i += nt) {
        if (restore) restore_one(b, i);
        if (zero) {
            set_p(b, i, 0.0);
            b.f_p[3 * i] = b.f_p[3 * i + 1] = b.f_p[3 * i + 2] = 0.f;
        }
        if (!is_ghost(b, i)) motion_one(p, b, i, dim);
    }
}

// set membership for one iteration (pcisph.py:634-643); row_mask bit n set
// when region n is scheduled; S_ob refreshed from the observed mask first
__global__ void __launch_bounds__(256) k_sets(const __grid_constant__ RtsParams p, RtsBuffers b,
                                              int row_mask, int all_pred) {
    RTS_ITER_GUARD();
    if (row_mask < 0) row_mask = b.ctl->row_mask;
    const int gen = b.ctl ? b.ctl->stamp : 0;
    const int nf = p.n_fluid;
    // every region scheduled (or a synchronous baseline): pred = force = all
    // fluid; the pair kernels then walk 0..nf-1 directly (no lists)
    // a local-phase entry decided by the previous control (ctl->snap_op == 1)
    // snapshots p, f_p of every fluid particle here (motion leaves them alone)
    if (b.ctl && b.ctl->snap_op == 1) {
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x) {
            b.snap_p[i] = b.xs[4 * i + 3];
            b.snap_fp[3 * i] = b.f_p[3 * i];
            b.snap_fp[3 * i + 1] = b.f_p[3 * i + 1];
            b.snap_fp[3 * i + 2] = b.f_p[3 * i + 2];
        }
    }
    const int all_mask = ((1 << (p.n_regions + 1)) - 1) & ~1;
    if (all_pred || (p.n_regions > 0 && (row_mask & all_mask) == all_mask)) {
        // (ghost rows are skipped by every pass and not counted)
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            b.ctr->n_pred = nf - p.n_ghost;
            b.ctr->n_force = nf - p.n_ghost;
            b.ctr->lists_all = 1;
        }
        return;
    }
    const int stride = gridDim.x * blockDim.x;
    if (b.ghost) {
        for (int base = blockIdx.x * blockDim.x; base < nf; base += stride) {
            const int i = base + threadIdx.x;
            bool pred = false, force = false;
            if (i < nf && !is_ghost(b, i)) {
                const bool sob = observed_block(b, b.fluid_cells[i], gen);
                const bool turn = all_pred || ((row_mask >> b.region[i]) & 1);
                const bool se = b.in_se[i] != 0;
                pred = turn || se || sob;
                force = turn || se;
                b.pflag[i] = force;
            }
            block_append2<256>(pred, i, b.active, &b.ctr->n_pred, force, i, b.list2,
                               &b.ctr->n_force);
        }
        return;
    }
    // four particles per thread (vector loads of cells / regions / S_e bits)
    const int ng = (nf + 3) / 4;
    for (int gb = blockIdx.x * blockDim.x; gb < ng; gb += stride) {
        const int g = gb + threadIdx.x;
        unsigned mp = 0u, mf = 0u;
        if (g < ng) {
            const int i0 = 4 * g;
            int cl[4];
            int8_t rg[4];
            uint8_t se[4];
            if (i0 + 3 < nf) {
                const int4 c4 = reinterpret_cast<const int4 *>(b.fluid_cells)[g];
                const char4 r4 = reinterpret_cast<const char4 *>(b.region)[g];
                const uchar4 s4 = reinterpret_cast<const uchar4 *>(b.in_se)[g];
                cl[0] = c4.x; cl[1] = c4.y; cl[2] = c4.z; cl[3] = c4.w;
                rg[0] = r4.x; rg[1] = r4.y; rg[2] = r4.z; rg[3] = r4.w;
                se[0] = s4.x; se[1] = s4.y; se[2] = s4.z; se[3] = s4.w;
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const bool in = i0 + q < nf;
                    cl[q] = in ? b.fluid_cells[i0 + q] : 0;
                    rg[q] = in ? b.region[i0 + q] : 0;
                    se[q] = in ? b.in_se[i0 + q] : 0;
                }
            }
            uint8_t pf[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const bool in = i0 + q < nf;
                const bool turn = all_pred || ((row_mask >> rg[q]) & 1);
                const bool s = se[q] != 0;
                const bool pred = in && (turn || s || observed_block(b, cl[q], gen));
                const bool force = in && (turn || s);
                pf[q] = force;
                mp |= (unsigned)pred << q;
                mf |= (unsigned)force << q;
            }
            if (i0 + 3 < nf) {
                reinterpret_cast<uchar4 *>(b.pflag)[g] = make_uchar4(pf[0], pf[1], pf[2], pf[3]);
            } else {
                for (int q = 0; q < 4 && i0 + q < nf; ++q) b.pflag[i0 + q] = pf[q];
            }
        }
        block_append4x2<256>(mp, mf, 4 * g, b.active, &b.ctr->n_pred, b.list2, &b.ctr->n_force);
    }
}

// S_ob = observed[fluid_cells] for every fluid particle (pcisph.py:537-542)
__global__ void k_sob(const __grid_constant__ RtsParams p, RtsBuffers b) {
    RTS_MINOR_GUARD();
    const int gen = b.ctl ? b.ctl->stamp : 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.n_fluid;
         i += gridDim.x * blockDim.x)
        b.in_sob[i] = observed_block(b, b.fluid_cells[i], gen);
}

// rho*, err over the pred list; p += delta (rho* - rho0) on force members.
// Granularity adapts to the list length: large lists run one particle per
// thread (neighbouring lanes share neighbours -> few L1 lines per warp
// load); short lists (the later, S_e-driven iterations) run an 8-lane group
// per particle so the launch still has enough independent loads in flight.
constexpr int kPG = 8;

// Grid of the per-particle passes: one thread per particle, or -- on scenes
// small enough that kPG lanes per particle fit the default grid cap -- kPG
// threads per particle, so the kernels' group paths (shorter dependent load
// chains per thread) serve latency-bound desk-scale runs.  Large scenes are
// unaffected (the cap binds).
static inline int pass_blocks(const RtsParams *p) {
    return rts_blocks((long long)p->n_fluid * kPG, kThreads, RTS_PAIR_CAP);
}

// the pair passes use no shared memory: ask for the largest L1 once
template <class K>
static inline void pair_carveout(K kernel) {
    if (RTS_PAIR_CARVEOUT >= 0)
        cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                             RTS_PAIR_CARVEOUT);
}


template <int LG, int CH = 8>
RTS_DEV void density_one(const RtsParams &p, const RtsBuffers &b, int i, int lane,
                         unsigned gmask) {
    RTS_CHECK_IDX(b.ctr, i, p.n_fluid, 401);
    if (is_ghost(b, i)) return;
    const XsRow *xsr = xs_rows(b);
    const XsRow a = ld_xs(xsr + i);  // own row: x* and the fp64 p of the last update
    const double xi = a.x, yi = a.y, zi = a.z;
    const int c = b.cnt[i];
    RTS_CHECK(b.ctr, 0 <= c && c <= p.width, 402);
    const int n_tot = p.n_fluid + p.n_bound;
    const int *row = b.nbr + i;  // entry q at row[q * S]: coalesced across lanes
    const size_t S = p.nbr_stride;
    double acc = 0.0;
    if (LG == 1 && RTS_DENS_PF) {
        // two-stage pipeline: table entries two chunks ahead, x* gathers one
        // chunk ahead of the chunk being summed
        int jn[CH];
        XsRow on[CH];
#pragma unroll
        for (int u = 0; u < CH; ++u)
            jn[u] = u < c ? rts_safe_idx(b.ctr, __ldcs(row + u * S), n_tot, 403, i) : i;
#pragma unroll
        for (int u = 0; u < CH; ++u) on[u] = ld_xs3(xsr + jn[u]);
#pragma unroll
        for (int u = 0; u < CH; ++u)
            jn[u] = CH + u < c ? rts_safe_idx(b.ctr, __ldcs(row + (CH + u) * S), n_tot, 403, i) : i;
        for (int q = 0; q < c; q += CH) {
            XsRow o[CH];
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                o[u] = on[u];
                on[u] = ld_xs3(xsr + jn[u]);
                jn[u] = q + 2 * CH + u < c
                            ? rts_safe_idx(b.ctr, __ldcs(row + (q + 2 * CH + u) * S), n_tot, 403, i)
                            : i;
            }
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                if (q + u < c)
                    acc = xadd(acc, poly6(dist2(xsub(xi, o[u].x), xsub(yi, o[u].y),
                                                xsub(zi, o[u].z)),
                                          p.h2, p.c_poly6));
            }
        }
    } else if (LG == 1) {
        // software-pipelined: the next chunk's table entries (mostly DRAM:
        // the tables exceed L2) are requested before this chunk's gathers
        int jn[CH];
#pragma unroll
        for (int u = 0; u < CH; ++u)
            jn[u] = u < c ? rts_safe_idx(b.ctr, __ldcs(row + u * S), n_tot, 403, i) : i;
        for (int q = 0; q < c; q += CH) {
            int j8[CH];
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                j8[u] = jn[u];
                jn[u] = q + CH + u < c ? __ldcs(row + (q + CH + u) * S) : i;
            }
            XsRow o[CH];
#pragma unroll
            for (int u = 0; u < CH; ++u) o[u] = ld_xs3(xsr + j8[u]);
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                if (q + u < c)
                    acc = xadd(acc, poly6(dist2(xsub(xi, o[u].x), xsub(yi, o[u].y),
                                                xsub(zi, o[u].z)),
                                          p.h2, p.c_poly6));
            }
        }
    } else {
        // RTS_LG_CH entries per lane in flight (same per-lane order)
        for (int q0 = lane; q0 < c; q0 += LG * RTS_LG_CH) {
            XsRow o[RTS_LG_CH];
#pragma unroll
            for (int u = 0; u < RTS_LG_CH; ++u) {
                const int q = q0 + u * LG;
                o[u] = ld_xs3(xsr + (q < c ? rts_safe_idx(b.ctr, row[q * S], n_tot, 403, i) : i));
            }
#pragma unroll
            for (int u = 0; u < RTS_LG_CH; ++u)
                if (q0 + u * LG < c)
                    acc = xadd(acc, poly6(dist2(xsub(xi, o[u].x), xsub(yi, o[u].y),
                                                xsub(zi, o[u].z)),
                                          p.h2, p.c_poly6));
        }
#pragma unroll
        for (int o = LG / 2; o > 0; o >>= 1) acc = xadd(acc, __shfl_xor_sync(gmask, acc, o, LG));
    }
    if (lane == 0) {
        const double rho = xmul(p.mass, acc);
        const double diff = xsub(rho, p.rho0);
        b.rho[i] = (float)rho;
        b.err[i] = diff > 0.0 ? xdiv(diff, p.rho0) : 0.0;
        if (!isfinite(rho)) atomicOr(&b.ctr->err_flags, RTS_ERR_NONFINITE);
        if (b.ctr->lists_all || b.pflag[i]) {
            double pr = xadd(a.p, xmul(p.delta, diff));
            pr = pr > 0.0 ? pr : 0.0;
            set_p(b, i, pr);
        }
    }
}

template <int CH, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_density(const __grid_constant__ RtsParams p,
                                                      RtsBuffers b) {
    RTS_ITER_GUARD();
    const bool all = b.ctr->lists_all;  // every fluid particle, particle order
    const int n = all ? p.n_fluid : b.ctr->n_pred;  // (all: ghost rows skipped inside)
    const int nthreads = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    if ((long long)n * kPG <= nthreads) {
        const int wl = threadIdx.x & 31, lane = wl & (kPG - 1);
        const unsigned gmask = ((1u << kPG) - 1u) << (wl & ~(kPG - 1));
        for (int t = tid / kPG; t < n; t += nthreads / kPG) {
            density_one<kPG>(p, b, all ? t : b.active[t], lane, gmask);
        }
    } else {
        for (int t = tid; t < n; t += nthreads) {
            density_one<1, CH>(p, b, all ? t : b.active[t], 0, 0u);
        }
    }
}

// S_e, S_e blocks, max err, sum rho* and any S_e over all fluid
// (pcisph.py:662, 421-430, 682-683).  Each block owns a fixed contiguous
// chunk (multiple of 4: double2/float4/uchar4 vector accesses) and sums it
// in a fixed tree; the last block to finish adds the block partials in
// index order -- the sum is deterministic and needs no further launch.
RTS_DEV void se_one(const RtsParams &p, const RtsBuffers &b, int i, double e, float rho,
                    int with_se, double thr, int gen, double &s, double &m, int &any,
                    uint8_t &flag) {
    const bool se = with_se && e > thr;
    flag = se;
    const bool ghost = is_ghost(b, i);
    if (se) {
        // ghost rows keep their S_e flag and block stamps, but any(S_e) is
        // the owners' to report (a ghost's err may be stale here)
        if (!ghost) any = 1;
        const int c = b.fluid_cells[i];
        if (atomicExch(&b.se_stamp[c], gen) != gen) {  // first S_e particle of block c
            const int nx = p.dims[0], ny = p.dims[1], nz = p.dims[2];
            const int cz = c % nz, cy = (c / nz) % ny, cx = c / (ny * nz);
            for (int ax = max(0, cx - 1); ax <= min(nx - 1, cx + 1); ++ax)
                for (int ay = max(0, cy - 1); ay <= min(ny - 1, cy + 1); ++ay) {
                    const int base = (ax * ny + ay) * nz;
                    for (int az = max(0, cz - 1); az <= min(nz - 1, cz + 1); ++az)
                        b.near_stamp[base + az] = gen;
                }
        }
    }
    if (ghost) return;  // reductions over owned particles (all-reduced)
    if (e > m) m = e;
    s = xadd(s, (double)rho);
}

__global__ void __launch_bounds__(256) k_se_reduce(const __grid_constant__ RtsParams p,
                                                   RtsBuffers b, int with_se) {
    RTS_ITER_GUARD();
    __shared__ double ssum[8], smax[8];
    __shared__ int sany[8];
    __shared__ bool last;
    const int nf = p.n_fluid;
    const double thr = xmul(0.5, p.eta_max);
    const int chunk = (((nf + gridDim.x - 1) / gridDim.x) + 3) & ~3;
    const int i0 = blockIdx.x * chunk, i1 = min(nf, i0 + chunk);
    const int gen = b.ctl ? b.ctl->stamp + 1 : 1;
    double s = 0.0, m = 0.0;
    int any = 0;
    for (int g = i0 + 4 * threadIdx.x; g < i1; g += 4 * blockDim.x) {
        if (g + 3 < i1) {
            const double2 e01 = *reinterpret_cast<const double2 *>(b.err + g);
            const double2 e23 = *reinterpret_cast<const double2 *>(b.err + g + 2);
            const float4 r = *reinterpret_cast<const float4 *>(b.rho + g);
            uchar4 f;
            se_one(p, b, g, e01.x, r.x, with_se, thr, gen, s, m, any, f.x);
            se_one(p, b, g + 1, e01.y, r.y, with_se, thr, gen, s, m, any, f.y);
            se_one(p, b, g + 2, e23.x, r.z, with_se, thr, gen, s, m, any, f.z);
            se_one(p, b, g + 3, e23.y, r.w, with_se, thr, gen, s, m, any, f.w);
            if (with_se) *reinterpret_cast<uchar4 *>(b.in_se + g) = f;
        } else {
            for (int i = g; i < i1; ++i) {
                uint8_t f;
                se_one(p, b, i, b.err[i], b.rho[i], with_se, thr, gen, s, m, any, f);
                if (with_se) b.in_se[i] = f;
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        s = xadd(s, __shfl_down_sync(0xffffffffu, s, o));
        m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
    }
    any = __any_sync(0xffffffffu, any);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        ssum[warp] = s;
        smax[warp] = m;
        sany[warp] = any;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // one atomic per block: same-address atomics serialise in L2
        double t = 0.0, bm = 0.0;
        int ba = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            t = xadd(t, ssum[w]);
            bm = fmax(bm, smax[w]);
            ba |= sany[w];
        }
        if (bm > 0.0)
            atomicMax(reinterpret_cast<unsigned long long *>(&b.ctr->max_err),
                      (unsigned long long)__double_as_longlong(bm));
        if (ba) atomicOr(&b.ctr->any_se, 1);
        b.partial[blockIdx.x] = t;
        __threadfence();
        last = atomicAdd(&b.ctr->blocks_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    double t = 0.0;  // fixed-order sum of the block partials
    for (int q = threadIdx.x; q < (int)gridDim.x; q += blockDim.x) t = xadd(t, __ldcg(b.partial + q));
    for (int o = 16; o > 0; o >>= 1) t = xadd(t, __shfl_down_sync(0xffffffffu, t, o));
    if (lane == 0) ssum[warp] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double u = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) u = xadd(u, ssum[w]);
        b.ctr->sum_rho = u;
        b.ctr->blocks_done = 0;
    }
}


// observed blocks (regions.py:110-125): occupied and (bordering a strictly
// smaller region, or bordering an S_e block without being one); -> block_tmp
__global__ void k_observed(const __grid_constant__ RtsParams p, RtsBuffers b, int with_se) {
    (void)with_se;  // the S_e part is stamp-based (k_se_reduce / observed_block)
    RTS_MINOR_GUARD();
    const int nx = p.dims[0], ny = p.dims[1], nz = p.dims[2];
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < p.n_cells;
         c += gridDim.x * blockDim.x) {
        const int8_t f = b.block_field[c];
        bool obs = false;
        if (f > 0) {
            const int cz = c % nz, cy = (c / nz) % ny, cx = c / (ny * nz);
            int8_t m = 127;
            for (int ax = max(0, cx - 1); ax <= min(nx - 1, cx + 1); ++ax)
                for (int ay = max(0, cy - 1); ay <= min(ny - 1, cy + 1); ++ay) {
                    const int base = (ax * ny + ay) * nz;
                    for (int az = max(0, cz - 1); az <= min(nz - 1, cz + 1); ++az) {
                        const int q = base + az;
                        if (q == c) continue;
                        const int8_t v = b.block_field[q];
                        if (v > 0 && v < m) m = v;
                    }
                }
            obs = (m < f);
        }
        b.block_tmp[c] = obs;
    }
}

// pressure forces at x* over the force list (pcisph.py:238-271); same
// adaptive granularity as k_density.
// One pair term of _pressure_forces (pcisph.py:255-268) in fp64:
// s = m^2 (p_i + p_j) / rho0^2 * c (h - r)^2 / r  (wall j: 2 p_i), f -= s x_ij,
// with K = m^2 c / rho0^2 and K p_i folded per particle and 1/r from an fp32
// estimate + one fp64 Newton step: ~1e-13 relative per term (18 fp64
// operations), so f_p keeps 1e-4 parity even where the pair terms cancel
// (|f_p| << sum |terms|), without making the pass FP64-bound.
template <class T>
RTS_DEV void pforce_pair(const RtsParams &p, double xi, double yi, double zi, double k_i,
                         double k_wall, double K, int i, int j, XsRow o, T &fx, T &fy, T &fz) {
    if (j == i) return;
    const double dx = xi - o.x, dy = yi - o.y, dz = zi - o.z;
    const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
    if (!(r2 > 0.0) || !(r2 < p.h2)) return;  // r <= 0 or r >= h
    const double y = rsqrt_nr(r2);
    const double d = fma(-r2, y, p.h);  // h - r
    const double kk = j < p.n_fluid ? fma(o.p, K, k_i) : k_wall;
    const double s = kk * d * d * y;
    fx = fma(-s, dx, fx);
    fy = fma(-s, dy, fy);
    fz = fma(-s, dz, fz);
}

template <int LG, int kPF = 4>
RTS_DEV void pforce_one(const RtsParams &p, const RtsBuffers &b, int i, int lane,
                        unsigned gmask) {
    if (is_ghost(b, i)) return;
    const XsRow *xsr = xs_rows(b);
    // K = m^2 c_spiky / rho0^2; K p_i, and 2 K p_i for wall neighbours
    const double K = xmul(xmul(xmul(p.mass, p.mass), p.c_spiky), xdiv(1.0, xmul(p.rho0, p.rho0)));
    const XsRow a = ld_xs(xsr + i);
    const unsigned long long pol = l2_keep_policy();
    const double xi = a.x, yi = a.y, zi = a.z;
    const double k_i = K * a.p, k_wall = 2.0 * k_i;
    const int c = b.cnt[i];
    RTS_CHECK(b.ctr, 0 <= c && c <= p.width, 404);
    const int n_tot = p.n_fluid + p.n_bound;
    const int *row = b.nbr + i;  // entry q at row[q * S]: coalesced across lanes
    const size_t S = p.nbr_stride;
    double fx = 0.0, fy = 0.0, fz = 0.0;
    if (LG == 1 && RTS_PFOR_PF) {
        // x* / p gathers one chunk ahead, table entries two chunks ahead
        int jn[kPF], jc[kPF];
        XsRow on[kPF];
#pragma unroll
        for (int u = 0; u < kPF; ++u)
            jc[u] = u < c ? rts_safe_idx(b.ctr, __ldcs(row + u * S), n_tot, 405, i) : i;
#pragma unroll
        for (int u = 0; u < kPF; ++u) on[u] = ld_xs_keep(xsr + jc[u], pol);
#pragma unroll
        for (int u = 0; u < kPF; ++u)
            jn[u] = kPF + u < c ? rts_safe_idx(b.ctr, __ldcs(row + (kPF + u) * S), n_tot, 405, i) : i;
        for (int q = 0; q < c; q += kPF) {
            int j4[kPF];
            XsRow o4[kPF];
#pragma unroll
            for (int u = 0; u < kPF; ++u) {
                j4[u] = jc[u];
                o4[u] = on[u];
                jc[u] = jn[u];
                on[u] = ld_xs_keep(xsr + jn[u], pol);
                jn[u] = q + 2 * kPF + u < c
                            ? rts_safe_idx(b.ctr, __ldcs(row + (q + 2 * kPF + u) * S), n_tot, 405, i)
                            : i;
            }
#pragma unroll
            for (int u = 0; u < kPF; ++u)
                if (q + u < c)
                    pforce_pair(p, xi, yi, zi, k_i, k_wall, K, i, j4[u], o4[u],
                                fx, fy, fz);
        }
    } else if (LG == 1) {
        int jn[kPF];  // software-pipelined table reads, as in density_one
#pragma unroll
        for (int u = 0; u < kPF; ++u) jn[u] = u < c ? __ldcs(row + u * S) : i;
        for (int q = 0; q < c; q += kPF) {
            int j4[kPF];
#pragma unroll
            for (int u = 0; u < kPF; ++u) {
                j4[u] = jn[u];
                jn[u] = q + kPF + u < c ? __ldcs(row + (q + kPF + u) * S) : i;
            }
            XsRow o4[kPF];
#pragma unroll
            for (int u = 0; u < kPF; ++u) o4[u] = ld_xs_keep(xsr + j4[u], pol);
#pragma unroll
            for (int u = 0; u < kPF; ++u)
                if (q + u < c)
                    pforce_pair(p, xi, yi, zi, k_i, k_wall, K, i, j4[u], o4[u],
                                fx, fy, fz);
        }
    } else {
        for (int q0 = lane; q0 < c; q0 += LG * RTS_LG_CH) {
            int j[RTS_LG_CH];
            XsRow o[RTS_LG_CH];
#pragma unroll
            for (int u = 0; u < RTS_LG_CH; ++u) {
                const int q = q0 + u * LG;
                j[u] = q < c ? rts_safe_idx(b.ctr, row[q * S], n_tot, 405, i) : i;
                o[u] = ld_xs(xsr + j[u]);
            }
#pragma unroll
            for (int u = 0; u < RTS_LG_CH; ++u)
                if (q0 + u * LG < c)
                    pforce_pair(p, xi, yi, zi, k_i, k_wall, K, i, j[u], o[u], fx, fy,
                                fz);
        }
#pragma unroll
        for (int o = LG / 2; o > 0; o >>= 1) {
            fx = xadd(fx, __shfl_xor_sync(gmask, fx, o, LG));
            fy = xadd(fy, __shfl_xor_sync(gmask, fy, o, LG));
            fz = xadd(fz, __shfl_xor_sync(gmask, fz, o, LG));
        }
    }
    if (lane == 0) {
        b.f_p[3 * i] = (float)fx;
        b.f_p[3 * i + 1] = (float)fy;
        b.f_p[3 * i + 2] = (float)fz;
    }
}

template <int CH, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_pforces(const __grid_constant__ RtsParams p,
                                                      RtsBuffers b) {
    RTS_ITER_GUARD();
    const bool all = b.ctr->lists_all;  // every fluid particle, particle order
    const int n = all ? p.n_fluid : b.ctr->n_force;  // (all: ghost rows skipped inside)
    const int nthreads = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    if ((long long)n * kPG <= nthreads) {
        const int wl = threadIdx.x & 31, lane = wl & (kPG - 1);
        const unsigned gmask = ((1u << kPG) - 1u) << (wl & ~(kPG - 1));
        for (int t = tid / kPG; t < n; t += nthreads / kPG) {
            const int i = all ? t : b.list2[t];
            if (!all && lane == 0) b.list3[t] = i;  // the next motion pass's list
            pforce_one<kPG>(p, b, i, lane, gmask);
        }
    } else {
        for (int t = tid; t < n; t += nthreads) {
            const int i = all ? t : b.list2[t];
            if (!all) b.list3[t] = i;
            pforce_one<1, CH>(p, b, i, 0, 0u);
        }
    }
}

// _integrate (pcisph.py:759-768) + validity countdown (pcisph.py:580-584)
// per-block max |v| and |f_ext + f_p| of one particle (k_block_maxima with
// add_fp, grid.cu), from the integrated velocity
RTS_DEV void block_maxima_one(const RtsBuffers &b, int c, const float *v, const float *fe,
                              const float *fp) {
    atomic_max_pos(&b.vmax[c], norm3(v[0], v[1], v[2]));
    const double fx = xadd((double)fe[0], (double)fp[0]), fy = xadd((double)fe[1], (double)fp[1]),
                 fz = xadd((double)fe[2], (double)fp[2]);
    atomic_max_pos(&b.fmax[c], xsqrt(dist2(fx, fy, fz)));
}

// the refresh culling bound: max coordinate displacement of this minor step
// (one atomic per warp; non-negative floats order as their bit patterns)
RTS_DEV void note_displacement(const RtsBuffers &b, int countdown, float dmax) {
    if (!countdown) return;
    for (int o = 16; o > 0; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    if ((threadIdx.x & 31) == 0 && dmax > 0.f)
        atomicMax(reinterpret_cast<unsigned *>(&b.ctr->disp_cur), __float_as_uint(dmax));
}

RTS_DEV void integrate_one(const RtsParams &p, const RtsBuffers &b, int i, int countdown,
                           int gen, double dim, float &dmax) {
    // S_ob from the final S_e generation (the public x* is the host's fp32
    // view of the xs rows, PcisphSolver.xstar)
    if (countdown) b.in_sob[i] = observed_block(b, b.fluid_cells[i], gen);
    float nx[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double f = xadd((double)b.force[3 * i + a], (double)b.f_p[3 * i + a]);
        double v = xadd((double)b.vel[3 * i + a], xmul(f, dim));
        const float x0 = b.pos[3 * i + a];
        double x = xadd((double)x0, xmul(v, p.dt));
        if (x < p.clamp_lo[a]) {
            x = p.clamp_lo[a];
            v = 0.0;
        } else if (x > p.clamp_hi[a]) {
            x = p.clamp_hi[a];
            v = 0.0;
        }
        b.pos[3 * i + a] = (float)x;
        b.vel[3 * i + a] = (float)v;
        nx[a] = (float)x;
        dmax = fmaxf(dmax, fabsf(nx[a] - x0));
    }
    if (countdown & 2) block_maxima_one(b, b.fluid_cells[i], &b.vel[3 * i], &b.force[3 * i],
                                        &b.f_p[3 * i]);
    if (countdown) {
        const int sl = rts_safe_idx(b.ctr, b.slot_of[i], b.ctr->n_sorted, 502, 0);
        reinterpret_cast<float4 *>(b.cpos)[sl] = make_float4(nx[0], nx[1], nx[2], __int_as_float(i));
        int v = b.validity[i] - 1;
        const bool expired = v <= 0;
        if (expired) {
            const int8_t r = b.region[i];
            v = kValidity[r < 0 ? 0 : (r > 4 ? 4 : r)];
        }
        b.validity[i] = v;
        b.compute[i] = expired;
    }
}

// _integrate (pcisph.py:759-768) + validity countdown (pcisph.py:580-584);
// four particles per thread with vector loads/stores when no ghost rows exist.
// countdown bit 0: validity countdown / S_ob / candidate copies (RTS minor
// steps); bit 1: also the per-block maxima of the mid-major marking
// (vmax / fmax zeroed beforehand), saving the separate k_block_maxima pass.
#ifndef RTS_INTEG_MINB
#define RTS_INTEG_MINB 3  // 80 registers: integrate + marking -6 us per major vs none (78 / 96), 4 spills more
#endif
#if RTS_INTEG_MINB > 0
#define RTS_INTEG_BOUNDS __launch_bounds__(256, RTS_INTEG_MINB)
#else
#define RTS_INTEG_BOUNDS
#endif
template <bool MAXIMA>
__global__ void RTS_INTEG_BOUNDS k_integrate(const __grid_constant__ RtsParams p, RtsBuffers b,
                                             int countdown) {
    RTS_MINOR_GUARD();
    const double dim = xmul(p.dt, p.inv_mass);
    const int gen = b.ctl ? b.ctl->stamp : 0;
    if (b.ctl && countdown && blockIdx.x == 0 && threadIdx.x == 0)
        b.ctl->stats[b.ctl->minor].t_looped = gtimer();
    // positions move: only cpos is kept current, the x / y / z copies go stale
    if (blockIdx.x == 0 && threadIdx.x == 0) b.ctr->soa_fresh = 0;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    const int nf = p.n_fluid;
    float dmax = 0.f;  // max |dx| of one coordinate (refresh culling bound)
    if (b.ghost || RTS_INTEG_1PT) {  // one particle per thread (the whole grid streams)
        for (int i = tid; i < nf; i += nt)
            if (!is_ghost(b, i)) integrate_one(p, b, i, countdown, gen, dim, dmax);
        note_displacement(b, countdown, dmax);
        return;
    }
    const int ng = nf / 4;
    for (int g = tid; g < ng; g += nt) {
        float fe[12], fp[12], v[12], x[12];
        load12(b.force, g, fe);
        load12(b.f_p, g, fp);
        load12(b.vel, g, v);
        load12(b.pos, g, x);
#pragma unroll
        for (int c = 0; c < 12; ++c) {
            const int a = c % 3;
            const double f = xadd((double)fe[c], (double)fp[c]);
            double vv = xadd((double)v[c], xmul(f, dim));
            double xx = xadd((double)x[c], xmul(vv, p.dt));
            if (xx < p.clamp_lo[a]) {
                xx = p.clamp_lo[a];
                vv = 0.0;
            } else if (xx > p.clamp_hi[a]) {
                xx = p.clamp_hi[a];
                vv = 0.0;
            }
            const float x0 = x[c];
            x[c] = (float)xx;
            v[c] = (float)vv;
            dmax = fmaxf(dmax, fabsf(x[c] - x0));
        }
        store12(b.pos, g, x);
        store12(b.vel, g, v);
        if (countdown) {
            const int4 cells = reinterpret_cast<const int4 *>(b.fluid_cells)[g];
            const int4 slots = reinterpret_cast<const int4 *>(b.slot_of)[g];
            int4 val = reinterpret_cast<const int4 *>(b.validity)[g];
            const char4 reg = reinterpret_cast<const char4 *>(b.region)[g];
            const int cl[4] = {cells.x, cells.y, cells.z, cells.w};
            const int nso = b.ctr->n_sorted;
            const int sl[4] = {rts_safe_idx(b.ctr, slots.x, nso, 503, 0),
                               rts_safe_idx(b.ctr, slots.y, nso, 503, 0),
                               rts_safe_idx(b.ctr, slots.z, nso, 503, 0),
                               rts_safe_idx(b.ctr, slots.w, nso, 503, 0)};
            int vl[4] = {val.x, val.y, val.z, val.w};
            const int rg[4] = {reg.x, reg.y, reg.z, reg.w};
            uint8_t sob[4], cmp[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (MAXIMA) block_maxima_one(b, cl[q], &v[3 * q], &fe[3 * q], &fp[3 * q]);
                sob[q] = observed_block(b, cl[q], gen);
                reinterpret_cast<float4 *>(b.cpos)[sl[q]] =
                    make_float4(x[3 * q], x[3 * q + 1], x[3 * q + 2], __int_as_float(4 * g + q));
                int vv = vl[q] - 1;
                const bool expired = vv <= 0;
                if (expired) vv = kValidity[rg[q] < 0 ? 0 : (rg[q] > 4 ? 4 : rg[q])];
                vl[q] = vv;
                cmp[q] = expired;
            }
            reinterpret_cast<int4 *>(b.validity)[g] = make_int4(vl[0], vl[1], vl[2], vl[3]);
            reinterpret_cast<uchar4 *>(b.compute)[g] = make_uchar4(cmp[0], cmp[1], cmp[2], cmp[3]);
            reinterpret_cast<uchar4 *>(b.in_sob)[g] = make_uchar4(sob[0], sob[1], sob[2], sob[3]);
        }
    }
    for (int i = 4 * ng + tid; i < nf; i += nt) integrate_one(p, b, i, countdown, gen, dim, dmax);
    note_displacement(b, countdown, dmax);
}

// _mark_timestep_updates (pcisph.py:718-755) in two passes.  Block part, per
// tile of blocks plus a one-block halo in shared memory: the required level
// of every halo block (assign_regions, regions.py:38-75, from the per-block
// maxima the integrator just formed) -> block_raw, and "violating" where it
// is below the current level; each occupied block of the tile then drops to
// min(own, lowest violating level over its 27-block neighbourhood) -> new
// field in block_tmp, changed mask in block_flag.
constexpr int kMX = 4, kMY = 8, kMZ = 32;
constexpr int kMHX = kMX + 2, kMHY = kMY + 2, kMHZ = kMZ + 2;
constexpr int kMHalo = kMHX * kMHY * kMHZ;
constexpr int kMPer = (kMHalo + 255) / 256;

__global__ void __launch_bounds__(256) k_mark_blocks(const __grid_constant__ RtsParams p,
                                                     RtsBuffers b) {
    RTS_MINOR_GUARD();
    __shared__ int8_t s_viol[kMHalo];  // required level where violating, else 127
    __shared__ int8_t s_cur[kMHalo];
    __shared__ uint8_t s_occ[kMHalo];
    const int nx = p.dims[0], ny = p.dims[1], nz = p.dims[2];
    const int tx = (nx + kMX - 1) / kMX, ty = (ny + kMY - 1) / kMY, tz = (nz + kMZ - 1) / kMZ;
    const double sound_bound = xdiv(xmul(p.lambda_v, p.block_size), p.sound_speed);
    const double rm = xmul(p.block_size, p.mass);
    for (int t = blockIdx.x; t < tx * ty * tz; t += gridDim.x) {
        const int bz = (t % tz) * kMZ, by = ((t / tz) % ty) * kMY, bx = (t / (tz * ty)) * kMX;
        int cell[kMPer], cnt[kMPer];
        int8_t cur[kMPer];
        double vm[kMPer], fm[kMPer];
#pragma unroll
        for (int u = 0; u < kMPer; ++u) {
            const int h = threadIdx.x + u * 256;
            const int hz = h % kMHZ, hy = (h / kMHZ) % kMHY, hx = h / (kMHZ * kMHY);
            const int cx = bx + hx - 1, cy = by + hy - 1, cz = bz + hz - 1;
            const bool in = h < kMHalo && cx >= 0 && cx < nx && cy >= 0 && cy < ny && cz >= 0 &&
                            cz < nz;
            cell[u] = in ? (cx * ny + cy) * nz + cz : -1;
            cnt[u] = in ? __ldg(b.cell_count + cell[u]) : 0;
            cur[u] = in ? b.block_field[cell[u]] : 0;
        }
#pragma unroll
        for (int u = 0; u < kMPer; ++u) {
            vm[u] = cnt[u] > 0 ? __ldg(b.vmax + cell[u]) : 0.0;
            fm[u] = cnt[u] > 0 ? __ldg(b.fmax + cell[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kMPer; ++u) {
            const int h = threadIdx.x + u * 256;
            if (h >= kMHalo) break;
            const bool occ = cnt[u] > 0;
            const int8_t raw = occ ? assign_from(p, vm[u], fm[u], sound_bound, rm) : 0;
            const int hz = h % kMHZ, hy = (h / kMHZ) % kMHY, hx = h / (kMHZ * kMHY);
            const bool interior = hx >= 1 && hx <= kMX && hy >= 1 && hy <= kMY && hz >= 1 &&
                                  hz <= kMZ;
            if (interior && cell[u] >= 0) b.block_raw[cell[u]] = raw;
            s_viol[h] = (occ && raw < cur[u] && cur[u] > 0) ? raw : (int8_t)127;
            s_cur[h] = cur[u];
            s_occ[h] = occ;
        }
        __syncthreads();
        for (int q = threadIdx.x; q < kMX * kMY * kMZ; q += blockDim.x) {
            const int iz = q % kMZ, iy = (q / kMZ) % kMY, ix = q / (kMZ * kMY);
            const int cx = bx + ix, cy = by + iy, cz = bz + iz;
            if (cx >= nx || cy >= ny || cz >= nz) continue;
            const int hc = ((ix + 1) * kMHY + iy + 1) * kMHZ + iz + 1;
            const int8_t c0 = s_cur[hc];
            int8_t nw = 0;
            if (s_occ[hc]) {
                int8_t spread = 127;  // out-of-grid halo blocks hold 127
#pragma unroll
                for (int dx = 0; dx < 3; ++dx)
#pragma unroll
                    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
                        for (int dz = 0; dz < 3; ++dz) {
                            const int8_t v = s_viol[((ix + dx) * kMHY + iy + dy) * kMHZ + iz + dz];
                            spread = v < spread ? v : spread;
                        }
                nw = c0 < spread ? c0 : spread;
            }
            const int c = (cx * ny + cy) * nz + cz;
            b.block_tmp[c] = nw;
            b.block_flag[c] = nw < c0;
        }
        __syncthreads();
    }
}

// particle part + apply: particles of changed blocks take the new level, a
// fresh validity and compute = 1; the new field replaces the old one (the
// particle loop reads block_tmp, so the two loops need no ordering)
__global__ void k_mark_particles(const __grid_constant__ RtsParams p, RtsBuffers b) {
    RTS_MINOR_GUARD();
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    for (int i = tid; i < p.n_fluid; i += nt) {
        const int c = b.fluid_cells[i];
        if (b.block_flag[c]) {
            const int8_t r = b.block_tmp[c];
            b.region[i] = r;
            b.compute[i] = 1;
            b.validity[i] = kValidity[r < 0 ? 0 : (r > 4 ? 4 : r)];
        }
    }
    for (int c = tid; c < p.n_cells; c += nt) b.block_field[c] = b.block_tmp[c];
}

__global__ void k_vel_max(const __grid_constant__ RtsParams p, RtsBuffers b) {
    double m = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.n_fluid;
         i += gridDim.x * blockDim.x) {
        const double v = norm3(b.vel[3 * i], b.vel[3 * i + 1], b.vel[3 * i + 2]);
        if (v > m) m = v;
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0)
        atomicMax(reinterpret_cast<unsigned long long *>(&b.ctr->fmax_bits),
                  (unsigned long long)__double_as_longlong(m));
}

// restore: 0 snapshot, 1 revert, -1 take ctl->snap_op (0 none, 1 snapshot, 2 revert)
__global__ void k_snapshot(const __grid_constant__ RtsParams p, RtsBuffers b, int restore) {
    if (restore < 0) {
        const int op = b.ctl->snap_op;
        if (op == 0 || fatal(b.ctr)) return;
        restore = op == 2;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.n_fluid;
         i += gridDim.x * blockDim.x) {
        if (!restore) {
            b.snap_p[i] = b.xs[4 * i + 3];
            b.snap_fp[3 * i] = b.f_p[3 * i];
            b.snap_fp[3 * i + 1] = b.f_p[3 * i + 1];
            b.snap_fp[3 * i + 2] = b.f_p[3 * i + 2];
        } else {
            set_p(b, i, b.snap_p[i]);
            b.f_p[3 * i] = b.snap_fp[3 * i];
            b.f_p[3 * i + 1] = b.snap_fp[3 * i + 1];
            b.f_p[3 * i + 2] = b.snap_fp[3 * i + 2];
        }
    }
}


// p = 0, f_p = 0 for all fluid at minor start (pcisph.py:570-571)
__global__ void k_zero_pressure(const __grid_constant__ RtsParams p, RtsBuffers b) {
    RTS_MINOR_GUARD();
    if (b.ctl && blockIdx.x == 0 && threadIdx.x == 0)
        b.ctl->stats[b.ctl->minor].t_refreshed = gtimer();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.n_fluid;
         i += gridDim.x * blockDim.x) {
        set_p(b, i, 0.0);
        b.f_p[3 * i] = 0.0f;
        b.f_p[3 * i + 1] = 0.0f;
        b.f_p[3 * i + 2] = 0.0f;
    }
}

__global__ void k_major_begin(RtsBuffers b) {
    RtsControl *c = b.ctl;
    c->stop_major = 0;
    c->done = 0;
    c->failed = 0;
    c->fail_kind = 0;
    for (int m = 0; m < RTS_MAX_MINOR; ++m) c->stats[m].iterations = -1;
}

RTS_DEV void add_row_iters(RtsControl *c, int minor, int row) {
    const int packed = c->row_counts[minor][row];
    for (int n = 1; n <= 4; ++n) c->riters[n] += (packed >> (4 * n)) & 0xF;
}

// state reset of _correct_scheduled (pcisph.py:618-631) + first row; S_e = {}
__global__ void k_minor_begin(RtsBuffers b, int minor, int sync_mode) {
    RtsControl *c = b.ctl;
    // reads first, then writes (one round trip, see k_control)
    const int stop = c->stop_major;
    const float disp_total = b.ctr->disp_total, disp_cur = b.ctr->disp_cur;
    const int row_mask0 = sync_mode ? 0 : c->row_masks[minor][0];
    const int packed0 = sync_mode ? 0 : c->row_counts[minor][0];
    const int stamp = c->stamp;
    c->skipped = stop;
    if (stop) {
        c->done = 1;
        return;
    }
    c->minor = minor;
    c->stats[minor].t_begin = gtimer();
    // refresh culling: the last minor step's displacement joins the bound
    b.ctr->disp_total = __fadd_ru(disp_total, disp_cur);
    b.ctr->disp_cur = 0.f;
    c->it = c->g_count = c->local_active = c->local_banned = c->local_run = 0;
    c->early = 0;
    c->done = 0;
    c->corrected = 0;
    c->forced = 0;
    for (int n = 0; n < 5; ++n) c->riters[n] = 0;
    c->motion_all = 1;
    c->snap_op = 0;
    c->stamp = stamp + 1;  // fresh S_e generation: S_e = {} (pcisph.py:618)
    c->prev_force = 0;
    b.ctr->n_pred = 0;
    b.ctr->n_force = 0;
    b.ctr->lists_all = 0;
    b.ctr->max_err = 0.0;
    b.ctr->any_se = 0;
    if (!sync_mode) {
        c->row_mask = row_mask0;
        // add_row_iters on the riters just zeroed above
        for (int n = 1; n <= 4; ++n) c->riters[n] = (packed0 >> (4 * n)) & 0xF;
    } else {
        c->row_mask = 0x1E;
    }
}

// Decisions after one correction iteration: pcisph.py:673-715 (scheduled,
// sync_mode = 0) or pcisph.py:457-468 (synchronous baselines, sync_mode = 1).
// Writes the next iteration's row / motion / snapshot ops, or ends the loop
// (cond handle of the enclosing CUDA-graph while node, if any).
__global__ void k_control(const __grid_constant__ RtsParams p, RtsBuffers b, int sync_mode,
                          unsigned long long cond_handle, int local_attempts, int iteration_cap,
                          int n_part) {
    (void)n_part;  // sum_rho: completed by k_se_reduce's last block (and all-reduced on ranks)
    if (threadIdx.x != 0) return;
    RtsControl *c = b.ctl;
    RtsCounters *ctr = b.ctr;
    // One thread on the critical path of every iteration.  Every read comes
    // first (they issue back to back: one memory round trip), then the
    // decisions on registers, then every write -- with read-modify-writes in
    // program order, in-order issue waited a full round trip per field.
    int done = c->done;
    int it = c->it, g_count = c->g_count, local_active = c->local_active;
    int local_banned = c->local_banned, local_run = c->local_run, early = c->early;
    int failed = c->failed, minor = c->minor, stamp = c->stamp;
    int local_entered = c->local_entered, local_reverted = c->local_reverted;
    long long corrected = c->corrected, forced = c->forced;
    const int n_rows_m = c->n_rows[minor < 0 ? 0 : minor];
    const int n_pred = ctr->n_pred, n_force = ctr->n_force, any_se = ctr->any_se;
    const int lists_all = ctr->lists_all;
    const unsigned err_flags = ctr->err_flags;
    const double max_err = ctr->max_err, sum_rho = ctr->sum_rho;
    const int n_all = p.n_global > 0 ? p.n_global : p.n_fluid;
    if (!done) {
        int snap_op = 0, motion_all = 0, fail_kind = 0, fail_g = 0, row_mask = 0;
        double fail_err = 0.0;
        it += 1;
        corrected += sync_mode ? n_all : n_pred;
        forced += sync_mode ? n_all : n_force;
        if (local_active) local_run += 1; else g_count += 1;
        const double mean = n_all ? sum_rho / (double)n_all : 0.0;
        double avg = n_all ? xsub(xdiv(mean, p.rho0), 1.0) : 0.0;
        avg = avg > 0.0 ? avg : 0.0;
        const bool converged = max_err < p.eta_max && avg < p.eta_avg;
        const bool was_failed = failed;
        if (err_flags & RTS_ERR_FATAL) {
            done = 1;
            failed = 1;
            fail_kind = (err_flags & RTS_ERR_NONFINITE) ? 1 : 4;
        } else if (sync_mode) {
            motion_all = 1;
            if (it >= 3 && converged) {
                done = 1;
            } else if (it > iteration_cap + 3) {
                done = 1;
                failed = 1;
                fail_kind = 3;
                fail_g = it;
                fail_err = max_err;
            }
        } else if (converged && it >= 3) {
            done = 1;
        } else if (!converged && it >= 3) {
            if (local_active) {
                if (local_run >= local_attempts) {
                    snap_op = 2;  // revert p, f_p to the entry snapshot
                    motion_all = 1;
                    local_active = 0;
                    local_banned = 1;
                    local_reverted += 1;
                }
            } else if (xmul(avg, 100.0) < p.rho_T && !local_banned && any_se) {
                local_active = 1;
                local_run = 0;
                snap_op = 1;
                local_entered += 1;
            }
            if (g_count > 6) early = 1;
            if (g_count > iteration_cap) {
                done = 1;
                failed = 1;
                fail_kind = 2;
                fail_g = g_count;
                fail_err = max_err;
            }
        }
        if (!done && !sync_mode) {
            if (!local_active) {
                const int r = g_count % n_rows_m;
                row_mask = c->row_masks[minor][r];
                const int packed = c->row_counts[minor][r];  // add_row_iters
                for (int n = 1; n <= 4; ++n) c->riters[n] += (packed >> (4 * n)) & 0xF;
            }
            c->row_mask = row_mask;  // 0 = local pass
        }
        if (lists_all) motion_all = 1;  // the force set was every particle
        // writes
        c->snap_op = snap_op;
        c->it = it;
        c->corrected = corrected;
        c->forced = forced;
        c->local_run = local_run;
        c->g_count = g_count;
        c->local_active = local_active;
        c->local_banned = local_banned;
        c->local_entered = local_entered;
        c->local_reverted = local_reverted;
        c->early = early;
        c->last_max_err = max_err;
        c->last_avg_err = avg;
        c->motion_all = motion_all;
        if (failed && !was_failed) {
            c->failed = 1;
            c->fail_kind = fail_kind;
            c->fail_g = fail_g;
            c->fail_err = fail_err;
        }
        if (failed) c->stop_major = 1;
        c->done = done;
        // hand-over to the next iteration: motion list length, fresh counts,
        // the S_e generation just written by k_se_reduce becomes current
        c->prev_force = n_force;
        c->stamp = stamp + 1;
        if (!done) {
            ctr->lists_all = 0;
            ctr->n_pred = 0;
            ctr->n_force = 0;
            ctr->max_err = 0.0;
            ctr->any_se = 0;
        }
    }
    if (cond_handle) cudaGraphSetConditional((cudaGraphConditionalHandle)cond_handle, done ? 0 : 1);
}

__global__ void k_minor_end(RtsBuffers b, int minor) {
    RtsControl *c = b.ctl;
    if (c->skipped) return;
    // reads first, then writes (one round trip, see k_control)
    const int it = c->it, n_refresh = b.ctr->n_compute, early = c->early, failed = c->failed;
    int riters[5];
    for (int n = 0; n < 5; ++n) riters[n] = c->riters[n];
    const long long corrected = c->corrected, forced = c->forced;
    const double max_err = c->last_max_err, avg_err = c->last_avg_err;
    RtsMinorStats &s = c->stats[minor];
    s.iterations = it;
    s.n_refresh = n_refresh;
    s.early = early;
    for (int n = 0; n < 5; ++n) s.riters[n] = riters[n];
    s.corrected = corrected;
    s.forced = forced;
    s.max_err = max_err;
    s.avg_err = avg_err;
    s.t_end = gtimer();
    if (early || failed) c->stop_major = 1;
}
// count_missing (grid.py:165-212): one block layer of the fresh audit grid
// `a` around the particle's current block; true neighbours (fp64) missing
// from the table row of the refresh particle
__global__ void k_audit(const __grid_constant__ RtsParams pa, RtsBuffers a, RtsBuffers b) {
    const int n = b.ctr->n_compute;
    const int nx = pa.dims[0], ny = pa.dims[1], nz = pa.dims[2];
    const float4 *cpos = reinterpret_cast<const float4 *>(a.cpos);
    long long lost = 0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int i = b.active[t];
        const double xi = b.pos[3 * i], yi = b.pos[3 * i + 1], zi = b.pos[3 * i + 2];
        const int cx = trunc_axis(xi, pa.origin[0], pa.inv_block, nx);
        const int cy = trunc_axis(yi, pa.origin[1], pa.inv_block, ny);
        const int cz = trunc_axis(zi, pa.origin[2], pa.inv_block, nz);
        const int *row = b.nbr + i;
        const size_t S = pa.nbr_stride;
        const int c = b.cnt[i];
        for (int ax = max(0, cx - 1); ax <= min(nx - 1, cx + 1); ++ax)
            for (int ay = max(0, cy - 1); ay <= min(ny - 1, cy + 1); ++ay) {
                const int base = (ax * ny + ay) * nz;
                const int k0 = a.starts[base + max(0, cz - 1)];
                const int k1 = a.starts[base + min(nz - 1, cz + 1) + 1];
                for (int k = k0; k < k1; ++k) {
                    const float4 o = cpos[k];
                    if (!(dist2(xsub(xi, (double)o.x), xsub(yi, (double)o.y),
                                xsub(zi, (double)o.z)) < pa.h2))
                        continue;
                    const int j = a.order[k];
                    bool found = false;
                    for (int q = 0; q < c; ++q)
                        if (row[q * S] == j) { found = true; break; }
                    if (!found) ++lost;
                }
            }
    }
    if (lost) atomicAdd((unsigned long long *)&b.ctr->missing, (unsigned long long)lost);
}

}  // namespace

extern "C" {

int rts_pci_audit(const RtsParams *pa, const RtsBuffers *a, const RtsBuffers *b, void *stream) {
    rts_note_launch(), k_audit<<<rts_blocks(pa->n_fluid, 128), 128, 0, (cudaStream_t)stream>>>(*pa, *a, *b);
    RTS_LAUNCH_CHECK();
    return 0;
}


int rts_pci_walls(const RtsParams *p, const RtsBuffers *b, void *stream) {
    if (p->n_bound <= 0) return 0;
    rts_note_launch(), k_xs_walls<<<rts_blocks(p->n_bound, 256), 256, 0, (cudaStream_t)stream>>>(*p, *b);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_gather(const RtsParams *p, const RtsBuffers *b, void *stream) {
    rts_note_launch(), k_gather<<<rts_blocks(p->n_fluid + p->n_bound, 256), 256, 0,
                                   (cudaStream_t)stream>>>(*p, *b);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_major_particles(const RtsParams *p, const RtsBuffers *b, void *stream) {
    rts_note_launch(), k_major_particles<<<rts_blocks(p->n_fluid, 256), 256, 0, (cudaStream_t)stream>>>(*p, *b);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_refresh(const RtsParams *p, const RtsBuffers *b, int all, int two_layer_r1,
                    void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(&b->ctr->n_compute, 0, sizeof(int), s);
    // one 256-slot chunk per CTA over every CSR slot (fluid and walls)
    rts_note_launch(), k_refresh_list<<<rts_blocks((long long)p->n_fluid + p->n_bound, 256,
                                                   RTS_RLIST_CAP), 256, 0, s>>>(*p, *b, all);
    RTS_LAUNCH_CHECK();
    rts_note_launch(), k_refresh<<<pass_blocks(p), kThreads, 0, s>>>(*p, *b, two_layer_r1);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_grid_search(const RtsParams *p, const RtsBuffers *b, const int8_t *layers, int n,
                    void *stream) {
    if (n <= 0) return 0;
    rts_note_launch(), k_search<<<rts_blocks(n, kThreads), kThreads, 0, (cudaStream_t)stream>>>(
        *p, *b, layers, n);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_motion(const RtsParams *p, const RtsBuffers *b, int all, void *stream) {
    rts_note_launch(), k_motion<<<rts_blocks(p->n_fluid, 256), 256, 0, (cudaStream_t)stream>>>(*p, *b, all);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_sets(const RtsParams *p, const RtsBuffers *b, int row_mask, int all_pred,
                 void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    // one trip of four particles per thread over the whole fluid
    rts_note_launch(), k_sets<<<rts_blocks(((long long)p->n_fluid + 3) / 4, 256, RTS_SETS_CAP), 256, 0, s>>>(
        *p, *b, row_mask, all_pred);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_density(const RtsParams *p, const RtsBuffers *b, void *stream) {
    const int nb = pass_blocks(p);
    cudaStream_t s = (cudaStream_t)stream;
    // 2-chunk gather pipeline, 64 registers: 8 CTAs of 128 threads per SM
    static bool once = (pair_carveout(k_density<RTS_DENS_CH, RTS_DENS_MINB>), true);
    (void)once;
    rts_note_launch(), k_density<RTS_DENS_CH, RTS_DENS_MINB><<<nb, kThreads, 0, s>>>(*p, *b);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_se_reduce(const RtsParams *p, const RtsBuffers *b, int with_se, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;

    int blocks = (p->n_fluid + 1023) / 1024;
    if (blocks > kRedBlocks) blocks = kRedBlocks;
    if (blocks < 1) blocks = 1;
    rts_note_launch(), k_se_reduce<<<blocks, 256, 0, s>>>(*p, *b, with_se);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_observed(const RtsParams *p, const RtsBuffers *b, int with_se, void *stream) {
    rts_note_launch(), k_observed<<<rts_blocks(p->n_cells, 256), 256, 0, (cudaStream_t)stream>>>(*p, *b, with_se);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_sob(const RtsParams *p, const RtsBuffers *b, void *stream) {
    rts_note_launch(), k_sob<<<rts_blocks(p->n_fluid, 256), 256, 0, (cudaStream_t)stream>>>(*p, *b);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_pforces(const RtsParams *p, const RtsBuffers *b, void *stream) {
    const int nb = pass_blocks(p);
    cudaStream_t s = (cudaStream_t)stream;
    static bool once = (pair_carveout(k_pforces<RTS_PFOR_CH, RTS_PFOR_MINB>), true);
    (void)once;
    rts_note_launch(), k_pforces<RTS_PFOR_CH, RTS_PFOR_MINB><<<nb, kThreads, 0, s>>>(*p, *b);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_integrate(const RtsParams *p, const RtsBuffers *b, int countdown, void *stream) {
    // four particles per thread without ghost rows, one with them
    const int nb = rts_blocks(b->ghost || !RTS_INTEG_GRID4 ? p->n_fluid : ((long long)p->n_fluid + 3) / 4,
                              256);
    cudaStream_t s = (cudaStream_t)stream;
    if (countdown & 2)
        rts_note_launch(), k_integrate<true><<<nb, 256, 0, s>>>(*p, *b, countdown);
    else
        rts_note_launch(), k_integrate<false><<<nb, 256, 0, s>>>(*p, *b, countdown);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_mark_updates(const RtsParams *p, const RtsBuffers *b, void *stream) {
    // required levels (block_raw) included: rts_block_levels(expand = 2)
    // before this call is not needed
    cudaStream_t s = (cudaStream_t)stream;
    const long long tiles = (long long)((p->dims[0] + kMX - 1) / kMX) *
                            ((p->dims[1] + kMY - 1) / kMY) * ((p->dims[2] + kMZ - 1) / kMZ);
    const int tb = (int)(tiles < 148 * 8 ? tiles : 148 * 8);
    rts_note_launch(), k_mark_blocks<<<tb, 256, 0, s>>>(*p, *b);
    rts_note_launch(), k_mark_particles<<<rts_blocks(p->n_fluid > p->n_cells ? p->n_fluid : p->n_cells,
                                                     256), 256, 0, s>>>(*p, *b);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_snapshot(const RtsParams *p, const RtsBuffers *b, int restore, void *stream) {
    rts_note_launch(), k_snapshot<<<rts_blocks(p->n_fluid, 256), 256, 0, (cudaStream_t)stream>>>(*p, *b, restore);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_vel_max(const RtsParams *p, const RtsBuffers *b, void *stream) {
    rts_note_launch(), k_vel_max<<<rts_blocks(p->n_fluid, 256, 148 * 8), 256, 0, (cudaStream_t)stream>>>(*p, *b);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_zero_pressure(const RtsParams *p, const RtsBuffers *b, void *stream) {
    rts_note_launch(), k_zero_pressure<<<rts_blocks(p->n_fluid, 256), 256, 0, (cudaStream_t)stream>>>(*p, *b);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_major_begin(const RtsParams *p, const RtsBuffers *b, void *stream) {
    (void)p;
    rts_note_launch(), k_major_begin<<<1, 1, 0, (cudaStream_t)stream>>>(*b);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_minor_begin(const RtsParams *p, const RtsBuffers *b, int minor, int sync_mode,
                        void *stream) {
    (void)p;
    rts_note_launch(), k_minor_begin<<<1, 1, 0, (cudaStream_t)stream>>>(*b, minor, sync_mode);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_minor_end(const RtsParams *p, const RtsBuffers *b, int minor, void *stream) {
    (void)p;
    rts_note_launch(), k_minor_end<<<1, 1, 0, (cudaStream_t)stream>>>(*b, minor);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_pci_control(const RtsParams *p, const RtsBuffers *b, int sync_mode,
                    unsigned long long cond_handle, int local_attempts, int iteration_cap,
                    void *stream);

// Second streams (and events) for the fork/join parts of a correction
// iteration (slot 0) and of a minor-step head (slot 1); they work inside a
// stream capture as well.  Separate slots because a head's side stream stays
// joined to the major graph's capture while the iterations are captured into
// the conditional bodies.
static void side_stream(int slot, cudaStream_t *side, cudaEvent_t **ev) {
    constexpr int kMaxDev = 16;  // per device: streams / events belong to one context
    static cudaStream_t st[kMaxDev][2] = {};
    static cudaEvent_t e[kMaxDev][2][2];
    int dev = 0;
    cudaGetDevice(&dev);
    dev = dev < kMaxDev ? dev : kMaxDev - 1;
    if (!st[dev][slot]) {
        cudaStreamCreateWithFlags(&st[dev][slot], cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&e[dev][slot][0], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&e[dev][slot][1], cudaEventDisableTiming);
    }
    *side = st[dev][slot];
    *ev = e[dev][slot];
}

// One correction iteration with device-side control (pcisph.py:633-715 or
// 446-468): motion, sets, density + pressure, S_e/reductions, observed,
// pressure forces, control, snapshot/revert.
int rts_pci_iteration(const RtsParams *p, const RtsBuffers *b, int sync_mode,
                      unsigned long long cond_handle, int local_attempts, int iteration_cap,
                      void *stream) {
    // DAG: {motion || sets} -> density -> {pforces || S_e reduction} -> control
    // (independent kernels on a side stream; also inside a graph capture)
    cudaStream_t s = (cudaStream_t)stream;
    cudaStream_t side;
    cudaEvent_t *ev;
    side_stream(0, &side, &ev);
    int rc;
    cudaEventRecord(ev[0], s);
    cudaStreamWaitEvent(side, ev[0], 0);
    if ((rc = rts_pci_sets(p, b, -1, sync_mode, side))) return rc;
    if ((rc = rts_pci_motion(p, b, -1, stream))) return rc;
    cudaEventRecord(ev[1], side);
    cudaStreamWaitEvent(s, ev[1], 0);
    if ((rc = rts_pci_density(p, b, stream))) return rc;
    cudaEventRecord(ev[0], s);
    cudaStreamWaitEvent(side, ev[0], 0);
    if ((rc = rts_pci_se_reduce(p, b, !sync_mode, side))) return rc;
    if ((rc = rts_pci_pforces(p, b, stream))) return rc;
    cudaEventRecord(ev[1], side);
    cudaStreamWaitEvent(s, ev[1], 0);
    return rts_pci_control(p, b, sync_mode, cond_handle, local_attempts, iteration_cap, stream);
}

int rts_pci_control(const RtsParams *p, const RtsBuffers *b, int sync_mode,
                    unsigned long long cond_handle, int local_attempts, int iteration_cap,
                    void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int n_part = 0;  // k_se_reduce's last block already summed the partials
    rts_note_launch(), k_control<<<1, 32, 0, s>>>(*p, *b, sync_mode, cond_handle, local_attempts,
                                                  iteration_cap, n_part);
    RTS_LAUNCH_CHECK();
    // the snapshot / revert it decides (ctl->snap_op) is applied by the next
    // iteration's k_sets / k_motion
    return 0;
}

// The minor step of RTS mode (pcisph.py:544-610) up to the correction loop,
// and its tail after the loop.
int rts_pci_minor_head(const RtsParams *p, const RtsBuffers *b, int minor, void *stream) {
    int rc;
    cudaStream_t s = (cudaStream_t)stream, side;
    cudaEvent_t *ev;
    side_stream(1, &side, &ev);
    if ((rc = rts_pci_minor_begin(p, b, minor, 0, stream))) return rc;
    // {refresh} || {S_e = empty, observed blocks}; p, f_p = 0 is folded into the first motion
    cudaEventRecord(ev[0], s);
    cudaStreamWaitEvent(side, ev[0], 0);
    cudaMemsetAsync(b->in_se, 0, (size_t)p->n_fluid, side);
    if ((rc = rts_pci_observed(p, b, 0, side))) return rc;
    if ((rc = rts_pci_refresh(p, b, 0, 1, stream))) return rc;  // p, f_p = 0: first motion
    cudaEventRecord(ev[1], side);
    cudaStreamWaitEvent(s, ev[1], 0);
    return 0;
}

int rts_pci_minor_tail(const RtsParams *p, const RtsBuffers *b, int minor, int last,
                       void *stream) {
    int rc;
    if (!last) {  // integrator + per-block maxima of the mid-major marking in one pass
        cudaStream_t s = (cudaStream_t)stream;
        cudaMemsetAsync(b->vmax, 0, sizeof(double) * (size_t)p->n_cells, s);
        cudaMemsetAsync(b->fmax, 0, sizeof(double) * (size_t)p->n_cells, s);
        if ((rc = rts_pci_integrate(p, b, 3, stream))) return rc;  // includes S_ob / x* refresh
        if ((rc = rts_pci_mark_updates(p, b, stream))) return rc;  // required levels included
    } else if ((rc = rts_pci_integrate(p, b, 1, stream))) {
        return rc;
    }
    return rts_pci_minor_end(p, b, minor, stream);
}

// ---- CUDA graphs -----------------------------------------------------------
static long long g_body_kernels = 0;

static int add_while_loop(cudaStream_t cs, const RtsParams *p, const RtsBuffers *b, int sync_mode,
                          int local_attempts, int iteration_cap) {
    cudaStreamCaptureStatus st;
    cudaGraph_t g;
    const cudaGraphNode_t *deps;
    size_t ndeps;
    cudaError_t e = cudaStreamGetCaptureInfo(cs, &st, nullptr, &g, &deps, &ndeps);
    if (e != cudaSuccess) return (int)e;
    cudaGraphConditionalHandle h;
    e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    if (e != cudaSuccess) return (int)e;
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    e = cudaGraphAddNode(&node, g, deps, ndeps, &np);
    if (e != cudaSuccess) return (int)e;
    cudaGraph_t body = np.conditional.phGraph_out[0];
    cudaStream_t bs;
    cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking);
    e = cudaStreamBeginCaptureToGraph(bs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) return (int)e;
    const long long before = rts_launch_count();
    int rc = rts_pci_iteration(p, b, sync_mode, (unsigned long long)h, local_attempts,
                               iteration_cap, bs);
    g_body_kernels = rts_launch_count() - before;
    cudaGraph_t out;
    e = cudaStreamEndCapture(bs, &out);
    cudaStreamDestroy(bs);
    if (rc) return rc;
    if (e != cudaSuccess) return (int)e;
    e = cudaStreamUpdateCaptureDependencies(cs, &node, 1, cudaStreamSetCaptureDependencies);
    return (int)e;
}

static int reset_counters(const RtsBuffers *b, cudaStream_t s) {
    return rts_counters_reset(b, s);
}

// Whole RTS major step (pcisph.py:482-505) or synchronous step
// (pcisph.py:376-419) as one graph: the correction loops are conditional
// while nodes driven by k_control, so a major step runs with no host round
// trip.  mode: 0 RTS major with n_minor minors, 1 synchronous step.
void *rts_pci_graph_create(const RtsParams *p, const RtsBuffers *b, int mode, int n_minor,
                           int local_attempts, int iteration_cap, int *err) {
    *err = 0;
    cudaStream_t cs;
    cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) { *err = (int)e; cudaStreamDestroy(cs); return nullptr; }
    int rc = 0;
    const long long count0 = rts_launch_count();
    g_body_kernels = 0;
    do {
        if ((rc = reset_counters(b, cs))) break;
        if ((rc = rts_pci_major_begin(p, b, cs))) break;
        if ((rc = rts_grid_keys(p, b, mode == 0, 1, cs))) break;
        if ((rc = rts_grid_sort(p, b, cs))) break;
        if (mode == 0) {
            // {candidate gather} || {levels, major particles}: independent after
            // the sort (gather: cpos / slot_of; levels: block fields, regions)
            cudaStream_t side = cs;
            cudaEvent_t *ev;
            if (RTS_MAJOR_FORK) side_stream(1, &side, &ev);
            if (RTS_MAJOR_FORK) {
                cudaEventRecord(ev[0], cs);
                cudaStreamWaitEvent(side, ev[0], 0);
            }
            if ((rc = rts_pci_gather(p, b, side))) break;
            if ((rc = rts_block_levels(p, b, 1, cs))) break;
            if ((rc = rts_pci_major_particles(p, b, cs))) break;
            if (RTS_MAJOR_FORK) {
                cudaEventRecord(ev[1], side);
                cudaStreamWaitEvent(cs, ev[1], 0);
            }
            for (int j = 0; j < n_minor && !rc; ++j) {
                if ((rc = rts_pci_minor_head(p, b, j, cs))) break;
                if ((rc = add_while_loop(cs, p, b, 0, local_attempts, iteration_cap))) break;
                rc = rts_pci_minor_tail(p, b, j, j == n_minor - 1, cs);
            }
        } else {
            if ((rc = rts_pci_gather(p, b, cs))) break;
            if ((rc = rts_pci_minor_begin(p, b, 0, 1, cs))) break;
            if ((rc = rts_pci_refresh(p, b, 1, 0, cs))) break;  // p, f_p = 0: first motion
            if ((rc = add_while_loop(cs, p, b, 1, local_attempts, iteration_cap))) break;
            if ((rc = rts_pci_integrate(p, b, 0, cs))) break;
            rc = rts_pci_minor_end(p, b, 0, cs);
        }
    } while (0);
    cudaGraph_t g = nullptr;
    e = cudaStreamEndCapture(cs, &g);
    cudaStreamDestroy(cs);
    if (rc || e != cudaSuccess) {
        *err = rc ? rc : (int)e;
        if (g) cudaGraphDestroy(g);
        return nullptr;
    }
    RtsGraph *rg = new RtsGraph;
    rg->graph = g;
    const int loops = mode == 0 ? n_minor : 1;
    rg->body_kernels = g_body_kernels;
    rg->static_kernels = rts_launch_count() - count0 - loops * g_body_kernels;
    e = cudaGraphInstantiate(&rg->exec, g, 0);
    if (e != cudaSuccess) {
        *err = (int)e;
        cudaGraphDestroy(g);
        delete rg;
        return nullptr;
    }
    return rg;
}

// kernel nodes of a graph: static ones (run once per launch) and those of one
// conditional-body iteration (run once per correction iteration)
int rts_graph_kernel_counts(void *graph, long long *static_kernels, long long *body_kernels) {
    RtsGraph *rg = (RtsGraph *)graph;
    *static_kernels = rg->static_kernels;
    *body_kernels = rg->body_kernels;
    return 0;
}

int rts_graph_launch(void *graph, void *stream) {
    RtsGraph *rg = (RtsGraph *)graph;
    return (int)cudaGraphLaunch(rg->exec, (cudaStream_t)stream);
}

void rts_graph_destroy(void *graph) {
    RtsGraph *rg = (RtsGraph *)graph;
    if (!rg) return;
    if (rg->exec) cudaGraphExecDestroy(rg->exec);
    if (rg->graph) cudaGraphDestroy(rg->graph);
    delete rg;
}

}  // extern "C"
