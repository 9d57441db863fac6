// Shared device helpers for librtssph (sm_100a).
//
// Parity-critical arithmetic (block keys, r^2 < h^2 membership, density and
// EOS sums, level classification) is fp64 with explicitly rounded, never
// fused operations (__dadd_rn / __dmul_rn / ...), in the operand order of
// the reference's Python/numba expressions, so that from a common fp32
// state the B200 results equal the reference's fp64 results exactly (or up
// to the final fp32 store).  The library is also compiled with
// --fmad=false as a second line of defence.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rts_sph.h"

#define RTS_DEV __device__ __forceinline__

namespace rts {

RTS_DEV double xadd(double a, double b) { return __dadd_rn(a, b); }
RTS_DEV double xsub(double a, double b) { return __dsub_rn(a, b); }
RTS_DEV double xmul(double a, double b) { return __dmul_rn(a, b); }
RTS_DEV double xdiv(double a, double b) { return __ddiv_rn(a, b); }
RTS_DEV double xsqrt(double a) { return __dsqrt_rn(a); }

// ((dx*dx + dy*dy) + dz*dz), the numba/numpy evaluation order.
RTS_DEV double dist2(double dx, double dy, double dz) {
    return xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz));
}

// poly6 W(r^2) = ((c*d)*d)*d, d = h2 - r2 (kernels.py:23-32)
RTS_DEV double poly6(double r2, double h2, double c) {
    const double d = xsub(h2, r2);
    if (d <= 0.0) return 0.0;
    return xmul(xmul(xmul(c, d), d), d);
}
// np.floor((x - origin) * inv_block), clipped to [0, n-1] (grid.py:248-250)
RTS_DEV int cell_axis(double x, double o, double inv, int n) {
    const double v = floor(xmul(xsub(x, o), inv));
    if (!(v >= 0.0)) return 0;  // also catches NaN (those rows are flagged anyway)
    if (v >= (double)(n - 1)) return n - 1;
    return (int)v;
}

RTS_DEV int cell_of(const RtsParams &p, double x, double y, double z) {
    const int cx = cell_axis(x, p.origin[0], p.inv_block, p.dims[0]);
    const int cy = cell_axis(y, p.origin[1], p.inv_block, p.dims[1]);
    const int cz = cell_axis(z, p.origin[2], p.inv_block, p.dims[2]);
    return (cx * p.dims[1] + cy) * p.dims[2] + cz;
}

// |v| = sqrt((x^2 + y^2) + z^2) in fp64 (np.linalg.norm(axis=1))
RTS_DEV double norm3(float x, float y, float z) {
    return xsqrt(dist2((double)x, (double)y, (double)z));
}

// L2 residency hint for gathered rows (x*, p): loads tagged evict_last stay in
// L2 while the streamed neighbour tables (loaded evict_first) pass through.
RTS_DEV unsigned long long l2_keep_policy() {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
RTS_DEV float4 ldg_keep(const float4 *ptr, unsigned long long pol) {
    float4 v;
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
        : "l"(ptr), "l"(pol));
    return v;
}

// ---- predicted-position rows of the PCISPH pair passes -------------------
// One 32-byte, 32-byte-aligned record per particle: fp64 x* (wall rows: the
// static position) and fp64 p -- the pressure solve's internal state, kept
// at the reference's precision (pcisph.py:202-271, 432-437): rho*, err and
// the pressure update from a common state then equal the reference's fp64
// results, instead of inheriting a 1e-7 rounding of x* or p that
// p = delta (rho* - rho0) and the pressure-force sums amplify where
// rho* ~ rho0 or the pair terms cancel.  The public p (RtsBuffers.pres) is
// its fp32 mirror.  A neighbour gather is a single 256-bit load (one L2
// sector) with no fp32 -> fp64 conversions.
struct __align__(32) XsRow {
    double x, y, z, p;
};

RTS_DEV XsRow xs_unpack(unsigned long long r0, unsigned long long r1, unsigned long long r2,
                        unsigned long long r3) {
    XsRow r;
    r.x = __longlong_as_double((long long)r0);
    r.y = __longlong_as_double((long long)r1);
    r.z = __longlong_as_double((long long)r2);
    r.p = __longlong_as_double((long long)r3);
    return r;
}
RTS_DEV XsRow ld_xs(const XsRow *ptr) {
    unsigned long long r0, r1, r2, r3;
    asm volatile("ld.global.v4.b64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(r0), "=l"(r1), "=l"(r2), "=l"(r3) : "l"(ptr));
    return xs_unpack(r0, r1, r2, r3);
}
RTS_DEV XsRow ld_xs_keep(const XsRow *ptr, unsigned long long pol) {
    unsigned long long r0, r1, r2, r3;
    asm volatile("ld.global.L2::cache_hint.v4.b64 {%0, %1, %2, %3}, [%4], %5;"
                 : "=l"(r0), "=l"(r1), "=l"(r2), "=l"(r3) : "l"(ptr), "l"(pol));
    return xs_unpack(r0, r1, r2, r3);
}
// x* only (the density pass): the p word is not brought into registers
#ifndef RTS_XS_KEEP
#define RTS_XS_KEEP 0  // density gathers tagged L2 evict-last (A/B)
#endif
RTS_DEV XsRow ld_xs3(const XsRow *ptr) {
    XsRow r;
#if RTS_XS_KEEP
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.L2::cache_hint.v4.f64 {%0, %1, %2, _}, [%3], %4;"
                 : "=d"(r.x), "=d"(r.y), "=d"(r.z) : "l"(ptr), "l"(pol));
#else
    asm volatile("ld.global.v4.f64 {%0, %1, %2, _}, [%3];"
                 : "=d"(r.x), "=d"(r.y), "=d"(r.z) : "l"(ptr));
#endif
    r.p = 0.0;
    return r;
}
RTS_DEV void st_xs(XsRow *ptr, double x, double y, double z, double p) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(ptr), "d"(x), "d"(y), "d"(z),
                 "d"(p)
                 : "memory");
}
// x* only (the prediction leaves p alone)
RTS_DEV void st_xs3(XsRow *ptr, double x, double y, double z) {
    asm volatile("st.global.v2.f64 [%0], {%1, %2};\n\tst.global.f64 [%0+16], %3;" ::"l"(ptr),
                 "d"(x), "d"(y), "d"(z)
                 : "memory");
}

// 32-byte fp64 records (one 256-bit access)
RTS_DEV void st_f64x4(double *ptr, double a, double b, double c, double d) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(ptr), "d"(a), "d"(b), "d"(c),
                 "d"(d)
                 : "memory");
}
RTS_DEV double4 ld_f64x4(const double *ptr) {
    double4 r;
    asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(ptr));
    return r;
}

// ---- packed fp32x2 arithmetic (sm_100: FADD2 / FMUL2 / FFMA2) ------------
#ifndef RTS_SOA
#define RTS_SOA 1  // neighbour searches on the x / y / z candidate copies (A/B: 0)
#endif
typedef unsigned long long f32x2;
RTS_DEV f32x2 f2_pack(float a, float b) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
RTS_DEV f32x2 f2_sub(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
RTS_DEV f32x2 f2_mul(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
RTS_DEV f32x2 f2_fma(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// Membership masks of the candidates [cb, cb + n) of the SoA copies (cx, cy,
// cz; n <= 32), candidates below k_lo excluded: bit u <-> candidate cb + u,
// `mem` = r^2 < h^2 (1 - 1e-5), `amb` = inside the +-1e-5 band (those take the
// exact fp64 test).  Four candidates per 128-bit load of each array (cb must
// be a multiple of 4; the arrays are padded past the last slot), two per
// packed fp32x2 operation; bits collected from the sign bits of
// r^2 - bound with one funnel shift each.
RTS_DEV void classify_soa(const float *cx, const float *cy, const float *cz, int cb, int n,
                          int k_lo, float fxi, float fyi, float fzi, float lo, float hi,
                          unsigned &mem_out, unsigned &amb_out) {
    const f32x2 P = f2_pack(fxi, fxi), Q = f2_pack(fyi, fyi), R = f2_pack(fzi, fzi);
    const f32x2 L = f2_pack(lo, lo), H = f2_pack(hi, hi);
    const ulonglong2 *X = reinterpret_cast<const ulonglong2 *>(cx + cb);
    const ulonglong2 *Y = reinterpret_cast<const ulonglong2 *>(cy + cb);
    const ulonglong2 *Z = reinterpret_cast<const ulonglong2 *>(cz + cb);
    unsigned mem = 0u, out = 0u;  // first candidate ends in the top bit
    for (int u = 0; u < n; u += 4) {
        const ulonglong2 x = X[u >> 2], y = Y[u >> 2], z = Z[u >> 2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const f32x2 ex = f2_sub(P, h ? x.y : x.x), ey = f2_sub(Q, h ? y.y : y.x),
                        ez = f2_sub(R, h ? z.y : z.x);
            const f32x2 r2 = f2_fma(ex, ex, f2_fma(ey, ey, f2_mul(ez, ez)));
            const f32x2 m = f2_sub(r2, L), o = f2_sub(H, r2);
            mem = __funnelshift_l((unsigned)m, mem, 1);
            mem = __funnelshift_l((unsigned)(m >> 32), mem, 1);
            out = __funnelshift_l((unsigned)o, out, 1);
            out = __funnelshift_l((unsigned)(o >> 32), out, 1);
        }
    }
    const int nr = (n + 3) & ~3;
    unsigned valid = n == 32 ? 0xffffffffu : ((1u << n) - 1u);
    if (k_lo > cb) valid &= ~((1u << (k_lo - cb)) - 1u);  // (k_lo - cb < 4)
    mem = (__brev(mem) >> (32 - nr)) & valid;
    out = (__brev(out) >> (32 - nr)) & valid;
    mem_out = mem;
    amb_out = valid & ~mem & ~out;
}


// 1/sqrt(r2) in fp64 from the fp32 estimate and one Newton step: relative
// error ~1e-13 (the estimate's 2^-22 squared), 5 fp64 operations instead of
// the ~12 of a full-precision rsqrt.  r2 must be a normal fp32 value.
RTS_DEV double rsqrt_nr(double r2) {
    const double y = (double)rsqrtf((float)r2);
    return y * fma(-0.5 * r2, y * y, 1.5);
}

// ---- checked builds ------------------------------------------------------
// -DRTS_CHECKED=1 range-checks every gathered / scattered index of the hot
// kernels (compute-sanitizer is unavailable on this GPU pool): a violation
// sets RTS_ERR_CHECK (fatal: later kernels stop, the host raises) and the
// first failing site.  Release builds compile the checks away.
#ifndef RTS_CHECKED
#define RTS_CHECKED 0
#endif
RTS_DEV void rts_check_fail(RtsCounters *c, int site) {
    atomicCAS(&c->check_site, 0, site);
    atomicOr(&c->err_flags, RTS_ERR_CHECK);
}
#define RTS_CHECK(ctr, cond, site)                                   \
    do {                                                            \
        if (RTS_CHECKED && !(cond)) rts::rts_check_fail((ctr), (site)); \
    } while (0)
// i in [0, n)
#define RTS_CHECK_IDX(ctr, i, n, site) RTS_CHECK(ctr, (unsigned)(i) < (unsigned)(n), site)
// an index about to be dereferenced: checked builds substitute `safe` for an
// out-of-range value (after flagging it) so the faulty access never happens
RTS_DEV int rts_safe_idx(RtsCounters *c, int i, int n, int site, int safe) {
    if (RTS_CHECKED && (unsigned)i >= (unsigned)n) {
        rts_check_fail(c, site);
        return safe;
    }
    return i;
}

// ---- exact neighbour membership ------------------------------------------
// The reference keeps j iff fp64 ((dx^2 + dy^2) + dz^2) < h^2 (grid.py:140-144).
// Candidates are first classified in fp32 with a +-1e-5 relative band around
// h^2 (fp32 rounding of r^2 is < 3e-7 relative), only in-band candidates take
// the exact fp64 test, kept out of line so the compiler cannot speculate the
// fp64 work into every candidate test.
static __device__ __noinline__ bool exact_neighbour(double h2, float fxi, float fyi, float fzi,
                                                    float ox, float oy, float oz) {
    return dist2(xsub((double)fxi, (double)ox), xsub((double)fyi, (double)oy),
                 xsub((double)fzi, (double)oz)) < h2;
}

struct Band {
    float lo, hi;
    double h2;
};

RTS_DEV Band make_band(double h2) {
    Band b;
    b.lo = (float)(h2 * (1.0 - 1e-5));
    b.hi = (float)(h2 * (1.0 + 1e-5));
    b.h2 = h2;
    return b;
}

RTS_DEV bool in_support(const Band &bd, float fxi, float fyi, float fzi, float4 o) {
    // any fp32 evaluation order is fine here: the band absorbs its rounding
    const float ex = __fsub_rn(fxi, o.x), ey = __fsub_rn(fyi, o.y), ez = __fsub_rn(fzi, o.z);
    const float r2f = __fmaf_rn(ex, ex, __fmaf_rn(ey, ey, __fmul_rn(ez, ez)));
    if (r2f > bd.hi) return false;
    if (r2f < bd.lo) return true;
    return exact_neighbour(bd.h2, fxi, fyi, fzi, o.x, o.y, o.z);
}

// max of non-negative doubles via their bit patterns (monotone for >= 0)
RTS_DEV void atomic_max_pos(double *addr, double v) {
    if (v > 0.0)  // NaN and 0 never raise a maximum (matches `if v > out[c]`)
        atomicMax(reinterpret_cast<unsigned long long *>(addr),
                  (unsigned long long)__double_as_longlong(v));
}

RTS_DEV long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Flags written by earlier kernels in the stream are visible at kernel start;
// a plain (L1-cacheable) load suffices -- no system-scope volatile load.
RTS_DEV bool fatal(const RtsCounters *c) { return c->err_flags & RTS_ERR_FATAL; }

// warp-aggregated append of `pred` lanes to list[*count]
RTS_DEV void warp_append(bool pred, int value, int *list, int *count) {
    const unsigned mask = __ballot_sync(0xffffffffu, pred);
    if (!mask) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(mask) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(count, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (pred) list[base + __popc(mask & ((1u << lane) - 1u))] = value;
}

// Block-aggregated append of up to two predicates per thread: one global
// atomic per block and list (the loop around it must be block-uniform).
// Within a block the output keeps thread order.
template <int NT>
RTS_DEV void block_append2(bool p0, int v0, int *list0, int *count0, bool p1, int v1,
                           int *list1, int *count1) {
    constexpr int NW = NT / 32;
    __shared__ int s_w0[NW], s_w1[NW], s_base[2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned m0 = __ballot_sync(0xffffffffu, p0);
    const unsigned m1 = __ballot_sync(0xffffffffu, p1);
    if (lane == 0) {
        s_w0[warp] = __popc(m0);
        s_w1[warp] = __popc(m1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int a = 0, c = 0;
        for (int w = 0; w < NW; ++w) {
            const int x = s_w0[w], y = s_w1[w];
            s_w0[w] = a;
            s_w1[w] = c;
            a += x;
            c += y;
        }
        s_base[0] = a && count0 ? atomicAdd(count0, a) : 0;
        s_base[1] = c && count1 ? atomicAdd(count1, c) : 0;
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    if (p0 && list0) list0[s_base[0] + s_w0[warp] + __popc(m0 & lt)] = v0;
    if (p1 && list1) list1[s_base[1] + s_w1[warp] + __popc(m1 & lt)] = v1;
    __syncthreads();  // shared slots are reused by the next loop trip
}

// float3 rows of 4 consecutive particles as 3 float4 (16-byte aligned)
RTS_DEV void load12(const float *a, int g, float v[12]) {
    const float4 *q = reinterpret_cast<const float4 *>(a) + 3 * g;
    const float4 x = q[0], y = q[1], z = q[2];
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
    v[8] = z.x; v[9] = z.y; v[10] = z.z; v[11] = z.w;
}
RTS_DEV void store12(float *a, int g, const float v[12]) {
    float4 *q = reinterpret_cast<float4 *>(a) + 3 * g;
    q[0] = make_float4(v[0], v[1], v[2], v[3]);
    q[1] = make_float4(v[4], v[5], v[6], v[7]);
    q[2] = make_float4(v[8], v[9], v[10], v[11]);
}

// Block-aggregated append of up to four items per thread to each of two
// lists: bit q of m0 / m1 appends base + q.  Output order is thread order,
// then bit order (ascending indices for contiguous groups); one global
// atomic per block and list.  The loop around it must be block-uniform.
template <int NT>
RTS_DEV void block_append4x2(unsigned m0, unsigned m1, int base, int *list0, int *count0,
                             int *list1, int *count1) {
    constexpr int NW = NT / 32;
    __shared__ int s_w0[NW], s_w1[NW], s_base[2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c0 = __popc(m0), c1 = __popc(m1);
    int x0 = c0, x1 = c1;  // inclusive warp scans
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y0 = __shfl_up_sync(0xffffffffu, x0, o), y1 = __shfl_up_sync(0xffffffffu, x1, o);
        if (lane >= o) {
            x0 += y0;
            x1 += y1;
        }
    }
    if (lane == 31) {
        s_w0[warp] = x0;
        s_w1[warp] = x1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int a = 0, c = 0;
        for (int w = 0; w < NW; ++w) {
            const int u = s_w0[w], v = s_w1[w];
            s_w0[w] = a;
            s_w1[w] = c;
            a += u;
            c += v;
        }
        s_base[0] = a ? atomicAdd(count0, a) : 0;
        s_base[1] = c ? atomicAdd(count1, c) : 0;
    }
    __syncthreads();
    int o0 = s_base[0] + s_w0[warp] + x0 - c0, o1 = s_base[1] + s_w1[warp] + x1 - c1;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if ((m0 >> q) & 1u) list0[o0++] = base + q;
        if ((m1 >> q) & 1u) list1[o1++] = base + q;
    }
    __syncthreads();  // shared slots are reused by the next loop trip
}

RTS_DEV int warp_count_add(bool pred, int *count) {
    const unsigned mask = __ballot_sync(0xffffffffu, pred);
    const int lane = threadIdx.x & 31;
    if (mask && lane == __ffs(mask) - 1) atomicAdd(count, __popc(mask));
    return __popc(mask);
}

// region id of an occupied block from its maxima (regions.py:38-75)
RTS_DEV int8_t assign_from(const RtsParams &p, double vmax, double fmax, double sound_bound,
                           double rm) {
    const double r = p.block_size;
    // lambda_f * sqrt(r*m / f_max); f_max == 0 -> inf (numpy divide)
    const double fb = xmul(p.lambda_f, xsqrt(xdiv(rm, fmax)));
    int8_t region = 1;
    for (int n = 2; n <= p.n_max; ++n) {
        const double dt_n = xmul((double)n, p.dt_base);
        if (p.use_sound && !(dt_n <= sound_bound)) break;
        bool ok = (region == n - 1);
        ok = ok && ((fmax == 0.0) || (dt_n <= fb));
        const double beta = p.betas[n];
        if (isfinite(beta)) ok = ok && (xdiv(xmul(dt_n, vmax), r) <= xmul(p.alpha, beta));
        if (ok) region = (int8_t)n;
    }
    return region;
}

}  // namespace rts

// kernel-launch counter (reported by bench.py as gpu_launches)
extern "C" void rts_note_launch(void);
extern "C" long long rts_launch_count(void);

// owned CUDA graph (rts_pci_graph_create / rts_wcsph_graph_create)
struct RtsGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    long long static_kernels = 0;  // kernel nodes outside conditional bodies
    long long body_kernels = 0;    // kernel nodes per conditional-body iteration
};

// launch helpers
static inline int rts_blocks(long long n, int threads, int cap = 148 * 32) {
    long long b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (int)b;
}

#define RTS_LAUNCH_CHECK() \
    do { cudaError_t e__ = cudaGetLastError(); if (e__ != cudaSuccess) return (int)e__; } while (0)
