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

// ctr scalars of this rank -> out[4] (fp64): max_err, any_se, sum_rho, n_pred
__global__ void k_ctl_publish(const RtsCounters *__restrict__ c, double *__restrict__ out) {
    out[0] = c->max_err;
    out[1] = (double)c->any_se;
    out[2] = c->sum_rho;
    out[3] = (double)c->n_pred;
}

// all-gathered (world, 4) -> ctr: MAX of max_err / any_se, SUM (rank order)
// of sum_rho / n_pred
__global__ void k_ctl_fold(RtsCounters *__restrict__ c, const double *__restrict__ g, int world) {
    double mx = g[0], se = g[1], sr = g[2], np_ = g[3];
    for (int r = 1; r < world; ++r) {
        const double *q = g + 4 * r;
        mx = fmax(mx, q[0]);
        se = fmax(se, q[1]);
        sr = __dadd_rn(sr, q[2]);
        np_ = __dadd_rn(np_, q[3]);
    }
    c->max_err = mx;
    c->any_se = (int32_t)se;
    c->sum_rho = sr;
    c->n_pred = (int32_t)np_;
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

}  // extern "C"
