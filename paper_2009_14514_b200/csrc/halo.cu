// Ghost-band pack / unpack and the per-iteration rank fold of the x-slab
// decomposition (distributed.py).
//
// The reference is single-process (pcisph.py:612-716 runs its correction
// loop over one particle set), so these entry points have no reference
// counterpart: they exist so that a rank's exchange of a phase is ONE pack
// launch, one grouped NCCL send/recv of a contiguous word buffer, and ONE
// unpack launch -- no per-field host indexing -- and so that the four
// convergence scalars of every correction iteration are folded across ranks
// on the device in rank order (deterministic) from a single all-gather.
//
// Messages are raw 32-bit words: fp64 fields travel as two words, so every
// exchanged value arrives bit-identical.
#include "common.cuh"

namespace {

constexpr int kThreads = 256;

// One thread per (row, field word): consecutive threads walk a row's words,
// so the message side is coalesced; the field side reads / writes rows[r]
// of each field, rows being sorted (global-id order), so neighbouring
// threads touch neighbouring storage rows.
template <bool kPack>
__global__ void __launch_bounds__(kThreads)
k_halo(const RtsHaloSpec s, const int32_t *__restrict__ rows, long long n,
       uint32_t *__restrict__ msg) {
    const long long total = n * s.row_words;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long r = t / s.row_words;
        int w = (int)(t - r * s.row_words);
        int f = 0;
        while (f < s.n_fields - 1 && w >= s.f[f].words) w -= s.f[f++].words;
        const RtsHaloField &fd = s.f[f];
        long long row = rows[r];
        if (row < 0) continue;  // padding entry (hole-filling plans)
        if (fd.remap) row = fd.remap[row];
        uint32_t *m = msg + r * s.msg_words + fd.msg_off + w;
        if (fd.esize == 1) {  // byte elements (int8 / bool fields): one per word
            uint8_t *p = (uint8_t *)fd.ptr + row * fd.stride + w;
            if (kPack) *m = *p;
            else *p = (uint8_t)*m;
        } else {
            uint32_t *p = (uint32_t *)fd.ptr + row * fd.stride + w;
            if (kPack) *m = *p;
            else *p = *m;
        }
    }
}

// ctr scalars of this rank -> out[5] (fp64): max_err, any_se, sum_rho,
// n_pred, err_flags (a uint32, exact in fp64)
__global__ void k_ctl_publish(const RtsCounters *__restrict__ c, double *__restrict__ out) {
    out[0] = c->max_err;
    out[1] = (double)c->any_se;
    out[2] = c->sum_rho;
    out[3] = (double)c->n_pred;
    out[4] = (double)c->err_flags;
}

// NaN-propagating max: a rank whose err went non-finite must stop every rank
RTS_DEV double nan_max(double a, double b) { return (a != a || b != b) ? a + b : fmax(a, b); }

// all-gathered (world, 5) -> ctr: MAX of max_err / any_se (NaN wins), SUM
// (rank order) of sum_rho / n_pred, OR of err_flags -- every rank then takes
// the same done / failed decision in k_control
__global__ void k_ctl_fold(RtsCounters *__restrict__ c, const double *__restrict__ g, int world) {
    double mx = g[0], se = g[1], sr = g[2], np_ = g[3];
    uint32_t fl = (uint32_t)g[4];
    for (int r = 1; r < world; ++r) {
        const double *q = g + RTS_CTL_WORDS * r;
        mx = nan_max(mx, q[0]);
        se = fmax(se, q[1]);
        sr = __dadd_rn(sr, q[2]);
        np_ = __dadd_rn(np_, q[3]);
        fl |= (uint32_t)q[4];
    }
    c->max_err = mx;
    c->any_se = (int32_t)se;
    c->sum_rho = sr;
    c->n_pred = (int32_t)np_;
    c->err_flags |= fl;
}

// Slab bookkeeping of a rank's owned rows [0, n) in one pass: block column
// bx = floor((x - origin_x) * inv_block) clipped to [0, nx) (the fp64
// expression of grid.py:248-250), then six row lists (order free: the grid
// sort orders block runs by global id):
//   0 / 1  migrants to the left / right neighbour (bx left the slab),
//   2 / 3  kept rows in the band of `halo` columns next to the left / right
//          neighbour (its ghosts),
//   4 / 5  migrants inside the neighbour's band next to this slab (they stay
//          here as ghosts: the neighbour would send them straight back);
// counts[6] = rows beyond a neighbour's slab (more than one slab per step).
__global__ void k_slab_classify(const RtsSlabGeom g, const float *__restrict__ pos, int n,
                                int32_t *__restrict__ lists, long long ls,
                                uint8_t *__restrict__ leave, int32_t *__restrict__ counts) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double v = floor(__dmul_rn(__dsub_rn((double)pos[3 * i], g.origin_x), g.inv_block));
        const int bx = !(v >= 0.0) ? 0 : (v >= (double)(g.nx - 1) ? g.nx - 1 : (int)v);
        uint8_t lv = 0;
        if (bx < g.lo) {
            if (!g.has_left || bx < g.left_lo) { atomicAdd(&counts[6], 1); continue; }
            lists[0 * ls + atomicAdd(&counts[0], 1)] = i;
            if (bx >= g.lo - g.halo) lists[4 * ls + atomicAdd(&counts[4], 1)] = i;
            lv = 1;
        } else if (bx >= g.hi) {
            if (!g.has_right || bx >= g.right_hi) { atomicAdd(&counts[6], 1); continue; }
            lists[1 * ls + atomicAdd(&counts[1], 1)] = i;
            if (bx < g.hi + g.halo) lists[5 * ls + atomicAdd(&counts[5], 1)] = i;
            lv = 1;
        } else {
            if (g.has_left && bx < g.lo + g.halo) lists[2 * ls + atomicAdd(&counts[2], 1)] = i;
            if (g.has_right && bx >= g.hi - g.halo) lists[3 * ls + atomicAdd(&counts[3], 1)] = i;
        }
        leave[i] = lv;
    }
}

// hole-filling plan: holes = leaving rows below n_keep, fill = kept rows at
// or above it (equal counts, paired in any order); the lists are pre-set to
// -1 (skipped by pack / unpack) up to the caller's bound
__global__ void k_slab_holes(const uint8_t *__restrict__ leave, int n, int n_keep,
                             int32_t *__restrict__ holes, int32_t *__restrict__ fill,
                             int32_t *__restrict__ counter) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (i < n_keep && leave[i]) holes[atomicAdd(&counter[0], 1)] = i;
        if (i >= n_keep && !leave[i]) fill[atomicAdd(&counter[1], 1)] = i;
    }
}

int check_spec(const RtsHaloSpec *s) {
    if (!s || s->n_fields < 1 || s->n_fields > RTS_HALO_MAX_FIELDS) return (int)cudaErrorInvalidValue;
    int words = 0;
    for (int f = 0; f < s->n_fields; ++f) {
        const RtsHaloField &fd = s->f[f];
        if (!fd.ptr || fd.words < 1 || fd.stride < fd.words || fd.msg_off < 0 ||
            (fd.esize != 0 && fd.esize != 1 && fd.esize != 4) ||
            fd.msg_off + fd.words > s->msg_words)
            return (int)cudaErrorInvalidValue;
        words += fd.words;
    }
    return words == s->row_words ? 0 : (int)cudaErrorInvalidValue;
}

template <bool kPack>
int launch_halo(const RtsHaloSpec *s, const int32_t *rows, int64_t n, uint32_t *msg,
                void *stream) {
    if (int rc = check_spec(s)) return rc;
    if (n <= 0) return 0;
    rts_note_launch();
    k_halo<kPack><<<rts_blocks(n * s->row_words, kThreads), kThreads, 0, (cudaStream_t)stream>>>(
        *s, rows, n, msg);
    RTS_LAUNCH_CHECK();
    return 0;
}

}  // namespace

extern "C" {

int rts_halo_pack(const RtsHaloSpec *s, const int32_t *rows, int64_t n, uint32_t *out,
                  void *stream) {
    return launch_halo<true>(s, rows, n, out, stream);
}

int rts_halo_unpack(const RtsHaloSpec *s, const int32_t *rows, int64_t n, const uint32_t *in,
                    void *stream) {
    return launch_halo<false>(s, rows, n, const_cast<uint32_t *>(in), stream);
}

int rts_ctl_publish(const RtsBuffers *b, double *out, void *stream) {
    rts_note_launch();
    k_ctl_publish<<<1, 1, 0, (cudaStream_t)stream>>>(b->ctr, out);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_ctl_fold(const RtsBuffers *b, const double *gathered, int world, void *stream) {
    if (world < 1) return (int)cudaErrorInvalidValue;
    rts_note_launch();
    k_ctl_fold<<<1, 1, 0, (cudaStream_t)stream>>>(b->ctr, gathered, world);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_slab_classify(const RtsSlabGeom *g, const float *pos, int n, int32_t *lists,
                      int64_t list_stride, uint8_t *leave, int32_t *counts, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(counts, 0, 8 * sizeof(int32_t), st);
    if (e != cudaSuccess) return (int)e;
    if (n <= 0) return 0;
    if (list_stride < n) return (int)cudaErrorInvalidValue;
    rts_note_launch();
    k_slab_classify<<<rts_blocks(n, kThreads), kThreads, 0, st>>>(*g, pos, n, lists, list_stride,
                                                                   leave, counts);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_slab_holes(const uint8_t *leave, int n, int n_keep, int n_pad, int32_t *holes,
                   int32_t *fill, int32_t *counter, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n_pad <= 0) return 0;
    cudaError_t e;
    if ((e = cudaMemsetAsync(holes, 0xff, (size_t)n_pad * 4, st)) != cudaSuccess) return (int)e;
    if ((e = cudaMemsetAsync(fill, 0xff, (size_t)n_pad * 4, st)) != cudaSuccess) return (int)e;
    if ((e = cudaMemsetAsync(counter, 0, 2 * sizeof(int32_t), st)) != cudaSuccess) return (int)e;
    rts_note_launch();
    k_slab_holes<<<rts_blocks(n, kThreads), kThreads, 0, st>>>(leave, n, n_keep, holes, fill,
                                                              counter);
    RTS_LAUNCH_CHECK();
    return 0;
}

}  // extern "C"
