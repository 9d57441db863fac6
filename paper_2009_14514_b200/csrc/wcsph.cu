// RTS-WCSPH step kernels (reference: /root/reference/pkg/src/rts_sph/wcsph.py).
//
// Neighbourhoods are never materialised: the density and force kernels walk
// the 3x3x3 block neighbourhood of each active particle directly in the CSR
// (the three z-adjacent blocks of each (x, y) column are one contiguous
// span, so nine spans), reading the sorted candidate copies `cpos`
// (x y z, p/rho^2 marker) and `cterm` (fp64 p/rho^2, 1/rho; v) written by the
// propagate pass.  The set of j
// with r^2 < h^2 (fp64, un-fused) and the visiting order (blocks in
// (ax, ay, az) order, CSR order inside a block) are exactly those of the
// reference's table fill (grid.py:133-149) followed by its table walk
// (wcsph.py:50-56, 75-101), so the fp64 sums are bit-identical to the
// reference's from a common state; only the final fp32 store rounds.
#include "common.cuh"

#ifndef RTS_WINT_GRID4
#define RTS_WINT_GRID4 1
#endif

// WCSPH force pass: table entries per gather chunk (1 = one at a time;
// scripts/build_variant.sh A/B)
#ifndef RTS_WF_CH
#define RTS_WF_CH 4
#endif

using namespace rts;

namespace {

constexpr int kThreads = 128;

#ifndef RTS_PROP_CTAS
#define RTS_PROP_CTAS 8  // propagate CTAs of 256 threads per SM (grid cap)
#endif

// 32-byte per-slot force-pass row: fp64 p/rho^2 and 1/rho of the slot's
// particle (this step's density for active slots, the stored state
// otherwise) and its fp32 velocity -- a neighbour is one 256-bit gather
// here plus its cpos row
struct TermRow {
    double term, inv_rho;
    float vx, vy, vz;
};
RTS_DEV void st_term(double *rows, int k, double term, double inv_rho, float vx, float vy,
                     float vz) {
    const unsigned long long v01 =
        (unsigned long long)__float_as_uint(vx) | ((unsigned long long)__float_as_uint(vy) << 32);
    const unsigned long long v2 = (unsigned long long)__float_as_uint(vz);
    asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(rows + 4 * (size_t)k),
                 "l"((unsigned long long)__double_as_longlong(term)),
                 "l"((unsigned long long)__double_as_longlong(inv_rho)), "l"(v01), "l"(v2)
                 : "memory");
}
RTS_DEV TermRow ld_term(const double *rows, int k) {
    unsigned long long r0, r1, r2, r3;
    asm volatile("ld.global.v4.b64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(r0), "=l"(r1), "=l"(r2), "=l"(r3) : "l"(rows + 4 * (size_t)k));
    TermRow t;
    t.term = __longlong_as_double((long long)r0);
    t.inv_rho = __longlong_as_double((long long)r1);
    t.vx = __uint_as_float((unsigned)(r2 & 0xffffffffull));
    t.vy = __uint_as_float((unsigned)(r2 >> 32));
    t.vz = __uint_as_float((unsigned)(r3 & 0xffffffffull));
    return t;
}

// wcsph.py:262-266 (validity / pre-emption) + sorted-copy gather + active list
__global__ void __launch_bounds__(256) k_propagate(const __grid_constant__ RtsParams p,
                                                   RtsBuffers b) {
    if (fatal(b.ctr)) return;
    if (!p.rts && blockIdx.x == 0 && threadIdx.x == 0) b.ctr->stamps[1] = gtimer();
    const int n_sorted = b.ctr->n_sorted;
    const int stride = gridDim.x * blockDim.x;
    for (int base = blockIdx.x * blockDim.x; base < n_sorted; base += stride) {
        const int k = base + threadIdx.x;
        bool act = false;
        if (k < n_sorted) {
            const int j = rts_safe_idx(b.ctr, b.order[k], p.n_fluid + p.n_bound, 201, 0);
            const float x = b.pos[3 * j], y = b.pos[3 * j + 1], z = b.pos[3 * j + 2];
            if (b.cx) b.cx[k] = x, b.cy[k] = y, b.cz[k] = z;
            if (j < p.n_fluid) {
                const double rho = b.rho[j], pr = b.pres[j];
                const double term = xdiv(pr, xmul(rho, rho)), inv_rho = xdiv(1.0, rho);
                reinterpret_cast<float4 *>(b.cpos)[k] = make_float4(x, y, z, (float)term);
                // the stored density / pressure of the slot's particle, fp64
                // (active particles overwrite them in the density pass)
                st_term(b.cterm, k, term, inv_rho, b.vel[3 * j], b.vel[3 * j + 1], b.vel[3 * j + 2]);
                if (p.rts) {
                    const int8_t blk = b.block_field[b.fluid_cells[j]];
                    int v = b.validity[j] - 1;
                    const int8_t reg = b.region[j];
                    act = (v <= 0) || (blk != reg);
                    if (act) {
                        b.region[j] = blk;
                        v = blk;
                    }
                    b.validity[j] = v;
                    b.compute[j] = act;
                } else {
                    act = true;
                }
            } else {
                reinterpret_cast<float4 *>(b.cpos)[k] = make_float4(x, y, z, -1.0f);
                st_term(b.cterm, k, 0.0, 0.0, 0.f, 0.f, 0.f);
            }
        }
        block_append2<256>(act, k, b.active, &b.ctr->n_compute, false, 0, nullptr, nullptr);
    }
}

struct Span {
    int k0, k1;
};

// the nine CSR spans of the 3x3x3 neighbourhood of block c, (ax, ay) order
__device__ __forceinline__ int block_spans(const RtsParams &p, const int *starts, int c,
                                           Span *sp) {
    const int nx = p.dims[0], ny = p.dims[1], nz = p.dims[2];
    const int cz = c % nz, cy = (c / nz) % ny, cx = c / (ny * nz);
    const int z0 = max(0, cz - 1), z1 = min(nz - 1, cz + 1);
    int n = 0;
    for (int ax = max(0, cx - 1); ax <= min(nx - 1, cx + 1); ++ax)
        for (int ay = max(0, cy - 1); ay <= min(ny - 1, cy + 1); ++ay) {
            const int base = (ax * ny + ay) * nz;
            sp[n].k0 = starts[base + z0];
            sp[n].k1 = starts[base + z1 + 1];
            ++n;
        }
    return n;
}

// ---- pair kernels -------------------------------------------------------
// The density pass walks the nine CSR spans with four float4 candidates in
// flight and collects the slots of true neighbours (exact reference
// membership, see in_support) into a per-thread shared-memory list, in
// reference order; it then evaluates the fp64 pair terms over that list
// without divergence and sums them sequentially in that order, so rho
// equals the reference's fp64 value from a common state (up to the fp32
// store).  The list is also kept in a column-major table (column = index in
// the active list, nbr[q * nbr_stride + t], cnt[t]), so the force pass of
// the same step reads its neighbours instead of searching again (positions
// do not change in between).
constexpr int kHitCap = 64;  // list entries per thread (overflow -> direct path)

RTS_DEV int collect_hits(const RtsParams &p, const RtsBuffers &b, const float4 *cpos, int cell,
                         float4 a, const Band &bd, int *hits, int *n_all) {
    // the nine column spans in (ax, ay) order, each one's starts requested
    // while the previous column is scanned (registers, not a local array);
    // columns outside the grid are empty spans
    const int nx = p.dims[0], ny = p.dims[1], nz = p.dims[2];
    const int cz = cell % nz, cy = (cell / nz) % ny, cx = cell / (ny * nz);
    const int z0 = max(0, cz - 1), z1 = min(nz - 1, cz + 1);
    auto span = [&](int s, int &k0, int &k1) {
        const int ax = cx + s / 3 - 1, ay = cy + s % 3 - 1;
        if (ax < 0 || ax >= nx || ay < 0 || ay >= ny) {
            k0 = k1 = 0;
            return;
        }
        const int base = (ax * ny + ay) * nz;
        k0 = b.starts[base + z0];
        k1 = b.starts[base + z1 + 1];
    };
    int nk0, nk1;
    span(0, nk0, nk1);
    int n = 0;
    for (int s = 0; s < 9; ++s) {
        const int k0 = nk0, k1 = nk1;
        if (s < 8) span(s + 1, nk0, nk1);
        // branch-free classification of 32 candidates at a time (sign bits of
        // r2 - bound collected with funnel shifts); in-band candidates take
        // the exact fp64 test; reads run up to 3 slots past the span (cpos
        // is padded)
        const bool soa = RTS_SOA && b.cx != nullptr;
        for (int cb = soa ? (k0 & ~3) : k0; cb < k1; cb += 32) {
            const int m = min(32, k1 - cb);
            const float4 *cp = cpos + cb;
            unsigned mem = 0u, out = 0u;
            if (soa) {  // x / y / z copies: 4 candidates per load, fp32x2 tests
                unsigned amb;
                classify_soa(b.cx, b.cy, b.cz, cb, m, k0, a.x, a.y, a.z, bd.lo, bd.hi, mem, amb);
                while (amb) {
                    const int q = __ffs(amb) - 1;
                    amb &= amb - 1u;
                    const float4 o = cp[q];
                    if (exact_neighbour(bd.h2, a.x, a.y, a.z, o.x, o.y, o.z)) mem |= 1u << q;
                }
            } else {
            for (int u = 0; u < m; u += 4) {
                float4 ob[4];
#pragma unroll
                for (int v = 0; v < 4; ++v) ob[v] = cp[u + v];
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const float ex = __fsub_rn(a.x, ob[v].x), ey = __fsub_rn(a.y, ob[v].y),
                                ez = __fsub_rn(a.z, ob[v].z);
                    const float r2f = __fmaf_rn(ex, ex, __fmaf_rn(ey, ey, __fmul_rn(ez, ez)));
                    mem = __funnelshift_l(__float_as_uint(__fsub_rn(r2f, bd.lo)), mem, 1);
                    out = __funnelshift_l(__float_as_uint(__fsub_rn(bd.hi, r2f)), out, 1);
                }
            }
            const int mr = (m + 3) & ~3;
            const unsigned valid = m == 32 ? 0xffffffffu : ((1u << m) - 1u);
            mem = (__brev(mem) >> (32 - mr)) & valid;
            out = (__brev(out) >> (32 - mr)) & valid;
            unsigned amb = valid & ~mem & ~out;
            while (amb) {
                const int q = __ffs(amb) - 1;
                amb &= amb - 1u;
                const float4 o = cp[q];
                if (exact_neighbour(bd.h2, a.x, a.y, a.z, o.x, o.y, o.z)) mem |= 1u << q;
            }
            }
            while (mem) {
                const int q = __ffs(mem) - 1;
                mem &= mem - 1u;
                if (n < kHitCap) hits[n * kThreads] = cb + q;
                ++n;
            }
        }
    }
    *n_all = n;
    return min(n, kHitCap);
}

// wcsph.py:45-60 over the on-the-fly search of grid.py:88-152
__global__ void __launch_bounds__(kThreads) k_density(const __grid_constant__ RtsParams p,
                                                      RtsBuffers b) {
    if (fatal(b.ctr)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) b.ctr->stamps[2] = gtimer();  // physics begins
    __shared__ int s_hits[kHitCap * kThreads];
    int *hits = s_hits + threadIdx.x;
    const int n_act = b.ctr->n_compute;
    const float4 *cpos = reinterpret_cast<const float4 *>(b.cpos);
    const Band bd = make_band(p.h2);
    const size_t S = p.nbr_stride;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_act; t += gridDim.x * blockDim.x) {
        const int k = rts_safe_idx(b.ctr, b.active[t], b.ctr->n_sorted, 202, 0);
        const int j = b.order[k];
        const float4 a = cpos[k];
        const double xi = a.x, yi = a.y, zi = a.z;
        int n_all;
        const int nh = collect_hits(p, b, cpos, b.fluid_cells[j], a, bd, hits, &n_all);
        b.cnt[t] = n_all;
        int *col = b.nbr + t;
        for (int q = 0; q < nh; ++q) col[q * S] = hits[q * kThreads];
        double acc = 0.0;
        if (n_all <= kHitCap) {
            for (int q = 0; q < nh; ++q) {
                const float4 o = cpos[hits[q * kThreads]];
                acc = xadd(acc, poly6(dist2(xsub(xi, (double)o.x), xsub(yi, (double)o.y),
                                            xsub(zi, (double)o.z)),
                                      p.h2, p.c_poly6));
            }
        } else {  // crowded neighbourhood: direct pass over the spans
            Span sp[9];
            const int ns = block_spans(p, b.starts, b.fluid_cells[j], sp);
            for (int s = 0; s < ns; ++s)
                for (int q = sp[s].k0; q < sp[s].k1; ++q)
                    if (in_support(bd, a.x, a.y, a.z, cpos[q])) {
                        const float4 o = cpos[q];
                        acc = xadd(acc, poly6(dist2(xsub(xi, (double)o.x), xsub(yi, (double)o.y),
                                                    xsub(zi, (double)o.z)),
                                              p.h2, p.c_poly6));
                    }
        }
        if (n_all > p.width) {
            atomicOr(&b.ctr->err_flags, RTS_ERR_OVERFLOW);
            atomicAdd((unsigned long long *)&b.ctr->overflow,
                      (unsigned long long)(n_all - p.width));
        }
        const double rho = xmul(p.mass, acc);
        const double ratio = xdiv(rho, p.rho0);
        const double r2 = xmul(ratio, ratio);
        const double r4 = xmul(r2, r2);
        double pr = xmul(p.b_stiff, xsub(xmul(xmul(ratio, r2), r4), 1.0));
        pr = pr > 0.0 ? pr : 0.0;
        if (!isfinite(rho)) atomicOr(&b.ctr->err_flags, RTS_ERR_NONFINITE);
        b.rho[j] = (float)rho;
        b.pres[j] = (float)pr;
        // publish p/rho^2 (wcsph.py:78, the reference's expression), 1/rho and
        // p in fp64 for the force pass: the pair terms then use this step's
        // fp64 density and pressure, as the reference does, not their fp32
        // stores (whose 6e-8 rounding the cancelling pair sums amplify)
        {
            const double term = xdiv(pr, xmul(rho, rho));
            st_term(b.cterm, k, term, xdiv(1.0, rho), b.vel[3 * j], b.vel[3 * j + 1],
                    b.vel[3 * j + 2]);
            // the wall pair term of this particle (wcsph.py:97): p/rho^2 + p/rho0^2
            b.cwall[k] = xadd(term, xmul(pr, xdiv(1.0, xmul(p.rho0, p.rho0))));
        }
    }
}

// One pair term of _forces (wcsph.py:75-101) in fp64, accumulated in the
// reference's neighbour order: with M = m^2 c_spiky and
// L_i = mu m^2 c_visc / rho_i folded per particle,
//   fluid j: F += L_i (h - r) / rho_j (v_j - v_i) - M (p_i/rho_i^2 + p_j/rho_j^2) (h - r)^2 / r x_ij
//   wall j:  F -= M (p_i/rho_i^2 + p_i/rho0^2) (h - r)^2 / r x_ij
// 1/r from an fp32 estimate + one fp64 Newton step: ~1e-13 relative per
// term, so the force keeps 1e-4 parity even where the pair terms cancel
// (hydrostatic rest: |F| << sum |terms|).
RTS_DEV void force_pair(const RtsParams &p, double xi, double yi, double zi, double vxi,
                        double vyi, double vzi, double L_i, double term_i, double wall_term,
                        double M, float4 o, TermRow tj, double &fx, double &fy, double &fz) {
    const double dx = xi - (double)o.x, dy = yi - (double)o.y, dz = zi - (double)o.z;
    const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
    if (!(r2 < p.h2)) return;                       // r >= h
    const double y = r2 > 0.0 ? rsqrt_nr(r2) : 0.0;  // r = 0: spiky 0, viscosity kept
    const double d = fma(-r2, y, p.h);              // h - r
    const double spk = M * d * d * y;               // m^2 c (h - r)^2 / r
    if (o.w >= 0.0f) {  // fluid neighbour: tj = (p_j / rho_j^2, 1 / rho_j in fp64; v_j)
        const double s = (term_i + tj.term) * spk;
        const double lap = L_i * d * tj.inv_rho;
        fx = fma(lap, (double)tj.vx - vxi, fma(-s, dx, fx));
        fy = fma(lap, (double)tj.vy - vyi, fma(-s, dy, fy));
        fz = fma(lap, (double)tj.vz - vzi, fma(-s, dz, fz));
    } else {  // static wall sample, mirrored pressure
        const double s = wall_term * spk;
        fx = fma(-s, dx, fx);
        fy = fma(-s, dy, fy);
        fz = fma(-s, dz, fz);
    }
}

// wcsph.py:288-296 + _forces wcsph.py:63-105
__global__ void __launch_bounds__(kThreads) k_forces(const __grid_constant__ RtsParams p,
                                                     RtsBuffers b) {
    if (fatal(b.ctr)) return;
    const size_t S = p.nbr_stride;
    const int n_act = b.ctr->n_compute;
    const float4 *cpos = reinterpret_cast<const float4 *>(b.cpos);
    const Band bd = make_band(p.h2);
    const double m2 = xmul(p.mass, p.mass);
    const double inv_rho0_sq = xdiv(1.0, xmul(p.rho0, p.rho0));
    const double M = xmul(m2, p.c_spiky), mum2c = xmul(xmul(p.mu, m2), p.c_visc);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_act; t += gridDim.x * blockDim.x) {
        const int k = b.active[t];
        const int j = b.order[k];
        const float4 a = cpos[k];
        const double xi = a.x, yi = a.y, zi = a.z;
        const TermRow own = ld_term(b.cterm, k);  // this step's fp64 p/rho^2, 1/rho; v
        const double term_i = own.term;
        const double L_i = mum2c * own.inv_rho;
        const double wall_term = b.cwall[k];
        const double vxi = own.vx, vyi = own.vy, vzi = own.vz;
        const int n_all = b.cnt[t];  // the density pass's neighbour list of slot k
        const int *col = b.nbr + t;
        double fx = 0.0, fy = 0.0, fz = 0.0;
        if (n_all <= kHitCap && RTS_WF_CH > 1) {
            // chunks of RTS_WF_CH entries: the chunk's table entries, then its
            // candidate gathers, are all in flight before its terms are
            // summed (same row order, so the same fp64 sums)
            for (int q0 = 0; q0 < n_all; q0 += RTS_WF_CH) {
                int kq[RTS_WF_CH];
                float4 pq[RTS_WF_CH];
                TermRow tq[RTS_WF_CH];
#pragma unroll
                for (int u = 0; u < RTS_WF_CH; ++u)
                    kq[u] = q0 + u < n_all
                                ? rts_safe_idx(b.ctr, col[(q0 + u) * S], b.ctr->n_sorted, 203, k)
                                : k;
#pragma unroll
                for (int u = 0; u < RTS_WF_CH; ++u) {
                    pq[u] = cpos[kq[u]];
                    tq[u] = ld_term(b.cterm, kq[u]);
                }
#pragma unroll
                for (int u = 0; u < RTS_WF_CH; ++u)
                    if (kq[u] != k)
                        force_pair(p, xi, yi, zi, vxi, vyi, vzi, L_i, term_i, wall_term, M, pq[u],
                                   tq[u], fx, fy, fz);
            }
        } else if (n_all <= kHitCap) {
            for (int q = 0; q < n_all; ++q) {
                const int kq = col[q * S];
                if (kq == k) continue;
                force_pair(p, xi, yi, zi, vxi, vyi, vzi, L_i, term_i, wall_term, M, cpos[kq],
                           ld_term(b.cterm, kq), fx, fy, fz);
            }
        } else {
            Span sp[9];
            const int ns = block_spans(p, b.starts, b.fluid_cells[j], sp);
            for (int s = 0; s < ns; ++s)
                for (int q = sp[s].k0; q < sp[s].k1; ++q)
                    if (q != k && in_support(bd, a.x, a.y, a.z, cpos[q]))
                        force_pair(p, xi, yi, zi, vxi, vyi, vzi, L_i, term_i, wall_term, M, cpos[q],
                                   ld_term(b.cterm, q), fx, fy, fz);
        }
        fx = xadd(fx, xmul(p.mass, p.gravity[0]));
        fy = xadd(fy, xmul(p.mass, p.gravity[1]));
        fz = xadd(fz, xmul(p.mass, p.gravity[2]));
        // bookkeeping of wcsph.py:288-290 for this active particle
        b.dt_corr[j] = b.dt_since[j];
        b.dt_since[j] = 0.0;
        float *ap = b.acc_prev + 3 * j;
        float *ac = b.acc + 3 * j;
        ap[0] = ac[0];
        ap[1] = ac[1];
        ap[2] = ac[2];
        float *fo = b.force + 3 * j;
        fo[0] = (float)fx;
        fo[1] = (float)fy;
        fo[2] = (float)fz;
        ac[0] = (float)xdiv(fx, p.mass);
        ac[1] = (float)xdiv(fy, p.mass);
        ac[2] = (float)xdiv(fz, p.mass);
    }
}

// wcsph.py:299-319: predictor for all, corrector (after it) for active, clamp
RTS_DEV void integrate_axis(const RtsParams &p, double dt, double half_dt2, bool correct,
                            double corr_x, double corr_v, int a, float &xf, float &vf, float acf,
                            float apf) {
    double x = xf, v = vf;
    const double ac = acf;
    x = xadd(x, xadd(xmul(v, dt), xmul(ac, half_dt2)));
    v = xadd(v, xmul(ac, dt));
    if (correct) {
        const double da = xsub(ac, (double)apf);
        x = xadd(x, xmul(da, corr_x));
        v = xadd(v, xmul(da, corr_v));
    }
    if (x < p.clamp_lo[a]) {
        x = p.clamp_lo[a];
        v = 0.0;
    } else if (x > p.clamp_hi[a]) {
        x = p.clamp_hi[a];
        v = 0.0;
    }
    xf = (float)x;
    vf = (float)v;
}

// four particles per thread with float4 / double2 vector accesses
__global__ void k_integrate(const __grid_constant__ RtsParams p, RtsBuffers b) {
    if (fatal(b.ctr)) return;
    const double dt = p.dt;
    const double half_dt2 = xmul(xmul(0.5, dt), dt);
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    const int nf = p.n_fluid, ng = nf / 4;
    for (int g = tid; g < ng; g += nt) {
        float x[12], v[12], ac[12], ap[12];
        load12(b.pos, g, x);
        load12(b.vel, g, v);
        load12(b.acc, g, ac);
        load12(b.acc_prev, g, ap);
        const double2 c01 = reinterpret_cast<const double2 *>(b.dt_corr)[2 * g];
        const double2 c23 = reinterpret_cast<const double2 *>(b.dt_corr)[2 * g + 1];
        double2 s01 = reinterpret_cast<const double2 *>(b.dt_since)[2 * g];
        double2 s23 = reinterpret_cast<const double2 *>(b.dt_since)[2 * g + 1];
        const uchar4 cm = reinterpret_cast<const uchar4 *>(b.compute)[g];
        const double dtc[4] = {c01.x, c01.y, c23.x, c23.y};
        const bool act[4] = {cm.x != 0, cm.y != 0, cm.z != 0, cm.w != 0};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const bool correct = p.apply_correction && (p.rts ? act[q] : true);
            const double corr_x = correct ? xdiv(xmul(dtc[q], dtc[q]), 6.0) : 0.0;
            const double corr_v = correct ? xdiv(dtc[q], 2.0) : 0.0;
#pragma unroll
            for (int a = 0; a < 3; ++a)
                integrate_axis(p, dt, half_dt2, correct, corr_x, corr_v, a, x[3 * q + a],
                               v[3 * q + a], ac[3 * q + a], ap[3 * q + a]);
        }
        store12(b.pos, g, x);
        store12(b.vel, g, v);
        s01.x = xadd(s01.x, dt);
        s01.y = xadd(s01.y, dt);
        s23.x = xadd(s23.x, dt);
        s23.y = xadd(s23.y, dt);
        reinterpret_cast<double2 *>(b.dt_since)[2 * g] = s01;
        reinterpret_cast<double2 *>(b.dt_since)[2 * g + 1] = s23;
    }
    for (int i = 4 * ng + tid; i < nf; i += nt) {
        const bool act = p.rts ? (b.compute[i] != 0) : true;
        const double dtc = b.dt_corr[i];
        const double corr_x = xdiv(xmul(dtc, dtc), 6.0);
        const double corr_v = xdiv(dtc, 2.0);
        const bool correct = p.apply_correction && act;
#pragma unroll
        for (int a = 0; a < 3; ++a)
            integrate_axis(p, dt, half_dt2, correct, corr_x, corr_v, a, b.pos[3 * i + a],
                           b.vel[3 * i + a], b.acc[3 * i + a], b.acc_prev[3 * i + a]);
        b.dt_since[i] = xadd(b.dt_since[i], dt);
    }
}

// np.var(rho) (wcsph.py:231-232, population variance over every fluid
// particle, stale entries included): two fixed-order passes -- the mean, then
// the mean squared deviation -- each a per-block fp64 tree over a fixed
// contiguous chunk, the block partials summed in block order by one thread.
// Deterministic; equals numpy's pairwise result to ~1e-16 relative.
constexpr int kVarBlocks = 256;

__global__ void __launch_bounds__(256) k_var_pass(const float *__restrict__ x, int n,
                                                  double *__restrict__ part, int second) {
    __shared__ double sh[256];
    const double mean = second ? part[2 * kVarBlocks] : 0.0;
    const int chunk = (n + gridDim.x - 1) / gridDim.x;
    const int i0 = blockIdx.x * chunk, i1 = min(n, i0 + chunk);
    double acc = 0.0;
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const double v = x[i];
        acc = xadd(acc, second ? xmul(xsub(v, mean), xsub(v, mean)) : v);
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] = xadd(sh[threadIdx.x], sh[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[second * kVarBlocks + blockIdx.x] = sh[0];
}

__global__ void k_var_fold(double *__restrict__ part, int n, int second, double *out) {
    double s = 0.0;
    for (int q = 0; q < kVarBlocks; ++q) s = xadd(s, part[second * kVarBlocks + q]);
    const double m = n > 0 ? xdiv(s, (double)n) : 0.0;
    if (!second) part[2 * kVarBlocks] = m;  // the mean, for the second pass
    else *out = m;
}

}  // namespace

extern "C" {

int rts_rho_variance(const RtsParams *p, const RtsBuffers *b, double *out, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    for (int second = 0; second < 2; ++second) {
        rts_note_launch(), k_var_pass<<<kVarBlocks, 256, 0, s>>>(b->rho, p->n_fluid, b->partial,
                                                                 second);
        RTS_LAUNCH_CHECK();
        rts_note_launch(), k_var_fold<<<1, 1, 0, s>>>(b->partial, p->n_fluid, second, out);
        RTS_LAUNCH_CHECK();
    }
    return 0;
}

int rts_wcsph_propagate(const RtsParams *p, const RtsBuffers *b, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(&b->ctr->n_compute, 0, sizeof(int), s);
    rts_note_launch(), k_propagate<<<rts_blocks(p->n_fluid + p->n_bound, 256, 148 * RTS_PROP_CTAS), 256, 0, s>>>(*p, *b);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_wcsph_density(const RtsParams *p, const RtsBuffers *b, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    rts_note_launch(), k_density<<<rts_blocks(p->n_fluid, kThreads), kThreads, 0, s>>>(*p, *b);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_wcsph_forces(const RtsParams *p, const RtsBuffers *b, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    rts_note_launch(), k_forces<<<rts_blocks(p->n_fluid, kThreads), kThreads, 0, s>>>(*p, *b);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_wcsph_integrate(const RtsParams *p, const RtsBuffers *b, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    // four particles per thread
    rts_note_launch(), k_integrate<<<rts_blocks(((long long)p->n_fluid + 3) / (RTS_WINT_GRID4 ? 4 : 1), 256),
                                     256, 0, s>>>(*p, *b);
    RTS_LAUNCH_CHECK();
    return 0;
}

// One RTS-WCSPH step (wcsph.py:199-233) captured as a CUDA graph: counters
// reset, rebuild, levels, propagate, density, forces, integrate.
void *rts_wcsph_graph_create(const RtsParams *p, const RtsBuffers *b, int *err) {
    *err = 0;
    cudaStream_t cs;
    cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) { *err = (int)e; cudaStreamDestroy(cs); return nullptr; }
    int rc = 0;
    const long long count0 = rts_launch_count();
    do {
        if ((rc = rts_counters_reset(b, cs))) break;
        if ((rc = rts_grid_keys(p, b, p->rts, 0, cs))) break;
        if ((rc = rts_grid_sort(p, b, cs))) break;
        if (p->rts && (rc = rts_block_levels(p, b, 0, cs))) break;
        if ((rc = rts_wcsph_propagate(p, b, cs))) break;
        if ((rc = rts_wcsph_density(p, b, cs))) break;
        if ((rc = rts_wcsph_forces(p, b, cs))) break;
        if ((rc = rts_wcsph_integrate(p, b, cs))) break;
        rc = rts_stamp(b, 3, cs);
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
    rg->static_kernels = rts_launch_count() - count0;
    e = cudaGraphInstantiate(&rg->exec, g, 0);
    if (e != cudaSuccess) {
        *err = (int)e;
        cudaGraphDestroy(g);
        delete rg;
        return nullptr;
    }
    return rg;
}

}  // extern "C"
