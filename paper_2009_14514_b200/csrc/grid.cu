// Block grid on the B200: keys, occupancy, boundary culling, stable counting
// sort into the CSR (starts, order) of the reference's BlockGrid
// (/root/reference/pkg/src/rts_sph/grid.py:220-394).
//
// Data layout (HBM): per-particle rows are canonical (reference index);
// per-block fields are dense over the padded grid dims, linearised
// (cx*ny + cy)*nz + cz (grid.py:252-255), so the three z-adjacent blocks of
// a 3x3x3 neighbourhood are contiguous in the CSR.
//
// Sort: fluid rows atomically bump their block count (integer, so
// deterministic); an exclusive scan gives `starts`; fluid rows scatter with
// an atomic cursor and each block's fluid run is then re-sorted by index,
// which restores the reference's stable order (fluid ascending, then active
// boundary ascending, grid.py:283-293) independent of atomic timing.
#include "common.cuh"

using namespace rts;

namespace {

constexpr int kThreads = 256;

// grid.py:257-277 (+ reduce_fluid_max, grid.py:155-162 / wcsph.py:239-240)
__global__ void k_fluid_keys(const __grid_constant__ RtsParams p, RtsBuffers b, int want_maxima,
                             int add_fp) {
    const int nf = p.n_fluid;
    const int stride = gridDim.x * blockDim.x;
    for (int base = blockIdx.x * blockDim.x; base < nf; base += stride) {
        const int i = base + threadIdx.x;
        if (i >= nf) break;
        const double x = b.pos[3 * i], y = b.pos[3 * i + 1], z = b.pos[3 * i + 2];
        const bool ok = (x >= p.origin[0]) && (x <= p.grid_hi[0]) && (y >= p.origin[1]) &&
                        (y <= p.grid_hi[1]) && (z >= p.origin[2]) && (z <= p.grid_hi[2]) &&
                        isfinite(x) && isfinite(y) && isfinite(z);
        if (!ok) {
            atomicOr(&b.ctr->err_flags, RTS_ERR_ESCAPED);
            atomicAdd(&b.ctr->n_escaped, 1);
            atomicMin(&b.ctr->first_escaped, i);
        }
        const int c = cell_of(p, x, y, z);
        b.fluid_cells[i] = c;
        atomicAdd(&b.cell_count[c], 1);
        if (want_maxima) {
            atomic_max_pos(&b.vmax[c], norm3(b.vel[3 * i], b.vel[3 * i + 1], b.vel[3 * i + 2]));
            double fx = b.force[3 * i], fy = b.force[3 * i + 1], fz = b.force[3 * i + 2];
            if (add_fp) {  // |f_ext + f_p| (pcisph.py:510), sum formed in fp64 like numpy
                fx = xadd(fx, (double)b.f_p[3 * i]);
                fy = xadd(fy, (double)b.f_p[3 * i + 1]);
                fz = xadd(fz, (double)b.f_p[3 * i + 2]);
                atomic_max_pos(&b.fmax[c], xsqrt(dist2(fx, fy, fz)));
            } else {
                atomic_max_pos(&b.fmax[c], xsqrt(dist2(fx, fy, fz)));
            }
        }
    }
}

__global__ void k_block_maxima(const __grid_constant__ RtsParams p, RtsBuffers b, int add_fp) {
    const int nf = p.n_fluid;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x) {
        const int c = b.fluid_cells[i];
        atomic_max_pos(&b.vmax[c], norm3(b.vel[3 * i], b.vel[3 * i + 1], b.vel[3 * i + 2]));
        double fx = b.force[3 * i], fy = b.force[3 * i + 1], fz = b.force[3 * i + 2];
        if (add_fp) {
            fx = xadd(fx, (double)b.f_p[3 * i]);
            fy = xadd(fy, (double)b.f_p[3 * i + 1]);
            fz = xadd(fz, (double)b.f_p[3 * i + 2]);
        }
        atomic_max_pos(&b.fmax[c], xsqrt(dist2(fx, fy, fz)));
    }
}

// boundary culling: a wall block participates iff a fluid particle occupies
// it or one of its 26 neighbours (dilate_mask(occupancy, 1), grid.py:279-290)
__global__ void k_boundary_active(const __grid_constant__ RtsParams p, RtsBuffers b) {
    if (fatal(b.ctr)) return;
    const int nx = p.dims[0], ny = p.dims[1], nz = p.dims[2];
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < p.n_bcells;
         t += gridDim.x * blockDim.x) {
        const int c = b.bcell_ids[t];
        const int cz = c % nz, cy = (c / nz) % ny, cx = c / (ny * nz);
        // the 27 counts requested together (no early exit: one round trip)
        int any = 0;
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx)
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                for (int dz = -1; dz <= 1; ++dz) {
                    const int ax = cx + dx, ay = cy + dy, az = cz + dz;
                    const bool in = ax >= 0 && ax < nx && ay >= 0 && ay < ny && az >= 0 && az < nz;
                    any |= in ? b.cell_count[(ax * ny + ay) * nz + az] : 0;
                }
        const bool allowed = any > 0;
        b.bcell_active[t] = allowed;
        b.cell_bcount[c] = allowed ? (b.bcell_start[t + 1] - b.bcell_start[t]) : 0;
    }
}

// ---- exclusive scan of (cell_count + cell_bcount) into starts ----------

__device__ __forceinline__ int block_incl_scan(int v, int *warp_sums) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    if (lane == 31) warp_sums[warp] = v;
    __syncthreads();
    if (warp == 0) {
        int s = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int n = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += n;
        }
        warp_sums[lane] = s;
    }
    __syncthreads();
    if (warp > 0) v += warp_sums[warp - 1];
    return v;
}

// Single-pass exclusive scan of cell_count + cell_bcount into starts with
// decoupled look-back: tiles take their index from an atomic counter (so a
// tile only waits on tiles that have started), publish their aggregate, then
// one warp walks back over the predecessors' status words (32 at a time)
// until it meets an inclusive prefix.  One launch instead of tile scan +
// recursive tile-sum scan + add + finish.
constexpr int kLbThreads = 256;
#ifndef RTS_SCAN_ITEMS
#define RTS_SCAN_ITEMS 16  // cells per thread (multiple of 4: int4 accesses)
#endif
constexpr int kLbItems = RTS_SCAN_ITEMS;
constexpr int kLbTile = kLbThreads * kLbItems;
constexpr unsigned long long kFlagAgg = 1ull << 32, kFlagPre = 2ull << 32;

__global__ void __launch_bounds__(kLbThreads) k_scan_lookback(const __grid_constant__ RtsParams p,
                                                              RtsBuffers b) {
    __shared__ int warp_sums[32];
    __shared__ int s_tile, s_excl;
    unsigned long long *status = reinterpret_cast<unsigned long long *>(b.scan_tmp + 2);
    int *counter = b.scan_tmp;
    const int n = p.n_cells;
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1);
    __syncthreads();
    const int tile = s_tile;
    const int i0 = tile * kLbTile + threadIdx.x * kLbItems;
    int v[kLbItems];
    int local = 0;
    const bool whole = i0 + kLbItems <= n;  // int4 accesses (i0 is a multiple of 4)
    if (whole) {
#pragma unroll
        for (int q = 0; q < kLbItems; q += 4) {
            const int4 a = *reinterpret_cast<const int4 *>(b.cell_count + i0 + q);
            const int4 w = *reinterpret_cast<const int4 *>(b.cell_bcount + i0 + q);
            v[q] = a.x + w.x, v[q + 1] = a.y + w.y, v[q + 2] = a.z + w.z, v[q + 3] = a.w + w.w;
            *reinterpret_cast<int4 *>(b.fill + i0 + q) = make_int4(0, 0, 0, 0);  // scatter cursors
        }
    } else {
#pragma unroll
        for (int q = 0; q < kLbItems; ++q) {
            const int idx = i0 + q;
            v[q] = idx < n ? b.cell_count[idx] + b.cell_bcount[idx] : 0;
            if (idx < n) b.fill[idx] = 0;
        }
    }
#pragma unroll
    for (int q = 0; q < kLbItems; ++q) local += v[q];
    const int incl = block_incl_scan(local, warp_sums);
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == kLbThreads - 1) {  // the tile's aggregate
        const unsigned long long word = (tile == 0 ? kFlagPre : kFlagAgg) | (unsigned)incl;
        __threadfence();
        atomicExch(status + tile, word);
        if (tile == 0) s_excl = 0;
    }
    if (tile > 0 && threadIdx.x < 32) {
        __syncwarp();
        int excl = 0, base = tile - 1;
        for (;;) {
            const int j = base - lane;
            unsigned long long w = kFlagPre;  // before tile 0: prefix 0
            if (j >= 0) {
                do {
                    w = atomicAdd(status + j, 0ull);
                } while ((w >> 32) == 0ull);
            }
            const bool pre = (w >> 32) == 2ull;
            const unsigned pm = __ballot_sync(0xffffffffu, pre);
            const int stop = pm ? __ffs(pm) - 1 : 31;  // nearest inclusive prefix
            int x = lane <= stop ? (int)(unsigned)(w & 0xffffffffull) : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            excl += x;
            if (pm) break;
            base -= 32;
        }
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    const int excl = s_excl;
    if (tile > 0 && threadIdx.x == kLbThreads - 1) {
        __threadfence();
        atomicExch(status + tile, kFlagPre | (unsigned)(excl + incl));
    }
    int run = excl + incl - local;
    if (whole) {
#pragma unroll
        for (int q = 0; q < kLbItems; q += 4) {
            int4 o;
            o.x = run, run += v[q];
            o.y = run, run += v[q + 1];
            o.z = run, run += v[q + 2];
            o.w = run, run += v[q + 3];
            *reinterpret_cast<int4 *>(b.starts + i0 + q) = o;
        }
    } else {
#pragma unroll
        for (int q = 0; q < kLbItems; ++q) {
            const int idx = i0 + q;
            if (idx < n) b.starts[idx] = run;
            run += v[q];
        }
    }
    if (i0 < n && i0 + kLbItems >= n) {  // owner of the last cell: total members
        b.starts[n] = run;
        b.ctr->n_sorted = run;
    }
}

// stable scatter, step 1: fluid rows take an atomic cursor in their block's
// run; the members of active wall blocks (threads past n_fluid) go straight
// to their static rank behind the fluid run (the wall CSR is sorted)
__global__ void k_scatter(const __grid_constant__ RtsParams p, RtsBuffers b) {
    if (fatal(b.ctr)) return;
    const int nf = p.n_fluid, nw = p.n_bcells > 0 ? p.n_bound : 0;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nf + nw;
         k += gridDim.x * blockDim.x) {
        if (k < nf) {
            const int c = b.fluid_cells[k];
            const int at = b.starts[c] + atomicAdd(&b.fill[c], 1);
            RTS_CHECK(b.ctr, at < b.starts[c] + b.cell_count[c], 101);
            b.order[rts_safe_idx(b.ctr, at, b.ctr->n_sorted, 102, 0)] = k;
        } else {
            const int q = k - nf;
            const int t = b.bcell_of[q];
            if (!b.bcell_active[t]) continue;
            const int c = b.bcell_ids[t];
            b.order[b.starts[c] + b.cell_count[c] + (q - b.bcell_start[t])] = b.bidx[q];
        }
    }
}

// step 2: restore ascending index order inside each block's fluid run.
// Runs of up to 16 (most WCSPH blocks, many PCISPH ones) are sorted in
// registers by a fully unrolled bitonic network (static indices, no local
// memory); runs up to 32 by insertion in a local array, longer ones in place.
#ifndef RTS_SORT_NET32
#define RTS_SORT_NET32 1  // runs of 17-32: bitonic network instead of insertion sort
#endif
RTS_DEV void cswap(int &a, int &b) {
    const int lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}
RTS_DEV void cswap(long long &a, long long &b) {
    const long long lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}
// ascending bitonic sorting network over N registers (N a power of two)
template <int N, class T>
RTS_DEV void bitonic(T (&v)[N]) {
#pragma unroll
    for (int k = 2; k <= N; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int q = 0; q < N; ++q) {
                const int r = q ^ j;
                if (r > q) {
                    if ((q & k) == 0) cswap(v[q], v[r]);
                    else cswap(v[r], v[q]);
                }
            }
}

__global__ void k_sort_runs(const __grid_constant__ RtsParams p, RtsBuffers b) {
    if (fatal(b.ctr)) return;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < p.n_cells;
         c += gridDim.x * blockDim.x) {
        const int n = b.cell_count[c];
        if (n < 2) continue;
        int *run = b.order + b.starts[c];
        if (n <= 16) {
            int v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = q < n ? run[q] : 0x7fffffff;
#pragma unroll
            for (int k = 2; k <= 16; k <<= 1)
#pragma unroll
                for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const int r = q ^ j;
                        if (r > q) {
                            if ((q & k) == 0) cswap(v[q], v[r]);
                            else cswap(v[r], v[q]);
                        }
                    }
#pragma unroll
            for (int q = 0; q < 16; ++q)
                if (q < n) run[q] = v[q];
        } else if (n <= 32) {  // 2.2-spacing blocks hold up to 27 lattice points
            int v[32];
#pragma unroll
            for (int q = 0; q < 32; ++q) v[q] = q < n ? run[q] : 0x7fffffff;
            if (RTS_SORT_NET32) {  // bitonic network: no data-dependent branches
#pragma unroll
                for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
                    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
                        for (int q = 0; q < 32; ++q) {
                            const int r = q ^ j;
                            if (r > q) {
                                if ((q & k) == 0) cswap(v[q], v[r]);
                                else cswap(v[r], v[q]);
                            }
                        }
            } else {
                for (int q = 1; q < n; ++q) {
                    const int key = v[q];
                    int r = q - 1;
                    while (r >= 0 && v[r] > key) { v[r + 1] = v[r]; --r; }
                    v[r + 1] = key;
                }
            }
#pragma unroll
            for (int q = 0; q < 32; ++q)
                if (q < n) run[q] = v[q];
        } else {
            for (int q = 1; q < n; ++q) {
                const int key = run[q];
                int r = q - 1;
                while (r >= 0 && run[r] > key) { run[r + 1] = run[r]; --r; }
                run[r + 1] = key;
            }
        }
    }
}

// x-slab ranks: fluid runs ordered by the rows' global ids (b.sort_key), so
// a rank's local row order is free while every within-block order -- and so
// every neighbour row and pair sum -- stays the single-domain one.
__global__ void k_sort_runs_keyed(const __grid_constant__ RtsParams p, RtsBuffers b) {
    if (fatal(b.ctr)) return;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < p.n_cells;
         c += gridDim.x * blockDim.x) {
        const int n = b.cell_count[c];
        if (n < 2) continue;
        int *run = b.order + b.starts[c];
        auto key = [&](int i) {
            return ((long long)b.sort_key[i] << 32) | (unsigned)i;
        };
        if (n <= 16) {  // (global id, row) keys through register bitonic networks
            long long v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = q < n ? key(run[q]) : 0x7fffffffffffffffll;
            bitonic<16>(v);
#pragma unroll
            for (int q = 0; q < 16; ++q)
                if (q < n) run[q] = (int)(v[q] & 0xffffffffll);
        } else if (n <= 32) {
            long long v[32];
#pragma unroll
            for (int q = 0; q < 32; ++q) v[q] = q < n ? key(run[q]) : 0x7fffffffffffffffll;
            bitonic<32>(v);
#pragma unroll
            for (int q = 0; q < 32; ++q)
                if (q < n) run[q] = (int)(v[q] & 0xffffffffll);
        } else {
            for (int q = 1; q < n; ++q) {
                const int x = run[q];
                const long long k = key(x);
                int r = q - 1;
                while (r >= 0 && key(run[r]) > k) { run[r + 1] = run[r]; --r; }
                run[r + 1] = x;
            }
        }
    }
}

__global__ void k_force_max(const __grid_constant__ RtsParams p, RtsBuffers b) {
    double m = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.n_fluid;
         i += gridDim.x * blockDim.x) {
        const double f = norm3(b.force[3 * i], b.force[3 * i + 1], b.force[3 * i + 2]);
        if (f > m) m = f;
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0)
        atomicMax(reinterpret_cast<unsigned long long *>(&b.ctr->fmax_bits),
                  (unsigned long long)__double_as_longlong(m));
}

__global__ void k_counters_reset(RtsCounters *c) {
    RtsCounters z = {};
    z.first_escaped = 0x7fffffff;
    z.stamps[0] = gtimer();
    *c = z;
}

__global__ void k_stamp(RtsCounters *c, int slot) { c->stamps[slot] = gtimer(); }

}  // namespace

extern "C" {

int rts_stamp(const RtsBuffers *b, int slot, void *stream) {
    rts_note_launch(), k_stamp<<<1, 1, 0, (cudaStream_t)stream>>>(b->ctr, slot);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_counters_reset(const RtsBuffers *b, void *stream) {
    rts_note_launch(), k_counters_reset<<<1, 1, 0, (cudaStream_t)stream>>>(b->ctr);
    RTS_LAUNCH_CHECK();
    return 0;
}


int rts_grid_keys(const RtsParams *p, const RtsBuffers *b, int want_maxima, int add_fp,
                  void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(b->cell_count, 0, sizeof(int) * (size_t)p->n_cells, s);
    if (want_maxima) {
        cudaMemsetAsync(b->vmax, 0, sizeof(double) * (size_t)p->n_cells, s);
        cudaMemsetAsync(b->fmax, 0, sizeof(double) * (size_t)p->n_cells, s);
    }
    rts_note_launch(), k_fluid_keys<<<rts_blocks(p->n_fluid, kThreads), kThreads, 0, s>>>(*p, *b, want_maxima,
                                                                        add_fp);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_block_maxima(const RtsParams *p, const RtsBuffers *b, int add_fp, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(b->vmax, 0, sizeof(double) * (size_t)p->n_cells, s);
    cudaMemsetAsync(b->fmax, 0, sizeof(double) * (size_t)p->n_cells, s);
    rts_note_launch(), k_block_maxima<<<rts_blocks(p->n_fluid, kThreads), kThreads, 0, s>>>(*p, *b, add_fp);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_grid_sort(const RtsParams *p, const RtsBuffers *b, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (p->n_bcells > 0) {
        rts_note_launch(), k_boundary_active<<<rts_blocks(p->n_bcells, kThreads), kThreads, 0, s>>>(*p, *b);
        RTS_LAUNCH_CHECK();
    }
    const int tiles = (p->n_cells + kLbTile - 1) / kLbTile;
    cudaMemsetAsync(b->scan_tmp, 0, sizeof(int) * (size_t)(2 + 2 * tiles), s);  // counter + status
    rts_note_launch(), k_scan_lookback<<<tiles, kLbThreads, 0, s>>>(*p, *b);
    RTS_LAUNCH_CHECK();
    rts_note_launch(), k_scatter<<<rts_blocks((long long)p->n_fluid + p->n_bound, kThreads), kThreads, 0, s>>>(
        *p, *b);
    RTS_LAUNCH_CHECK();
    if (b->sort_key)
        rts_note_launch(), k_sort_runs_keyed<<<rts_blocks(p->n_cells, kThreads), kThreads, 0, s>>>(*p, *b);
    else
        rts_note_launch(), k_sort_runs<<<rts_blocks(p->n_cells, kThreads), kThreads, 0, s>>>(*p, *b);
    RTS_LAUNCH_CHECK();
    return 0;
}

int rts_force_max(const RtsParams *p, const RtsBuffers *b, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    rts_note_launch(), k_force_max<<<rts_blocks(p->n_fluid, kThreads, 148 * 8), kThreads, 0, s>>>(*p, *b);
    RTS_LAUNCH_CHECK();
    return 0;
}

static unsigned long long g_launches = 0;
void rts_note_launch(void) { __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED); }
long long rts_launch_count(void) { return (long long)__atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int rts_abi_version(void) { return RTS_ABI_VERSION; }

int rts_device_sms(void) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return -(int)e;
    int sms = 0;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return -(int)e;
    return sms;
}

int rts_memset(void *dst, int value, int64_t bytes, void *stream) {
    return (int)cudaMemsetAsync(dst, value, (size_t)bytes, (cudaStream_t)stream);
}

}  // extern "C"
