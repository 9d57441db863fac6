// Region fields on the B200 (reference: /root/reference/pkg/src/rts_sph/regions.py).
//
// assign_regions (regions.py:38-75) is evaluated per block in fp64 with the
// reference's operation order, so levels are bit-identical given the same
// per-block maxima.  smooth_regions (regions.py:78-91) is a 26-neighbour min
// stencil; expand_fast_regions (regions.py:94-107) is a Chebyshev-4
// dilation done as three separable width-9 passes over a 2-bit mask.
#include "common.cuh"

using namespace rts;

namespace {

constexpr int kThreads = 256;
constexpr int8_t kEmpty = 127;  // regions.py:35

RTS_DEV int8_t assign_cell(const RtsParams &p, const RtsBuffers &b, int c, double sound_bound,
                           double rm) {
    if (b.cell_count[c] <= 0) return 0;
    return assign_from(p, b.vmax[c], b.fmax[c], sound_bound, rm);
}

__global__ void k_assign(const __grid_constant__ RtsParams p, RtsBuffers b) {
    if (fatal(b.ctr)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) b.ctr->stamps[1] = gtimer();  // grid rebuilt
    const double sound_bound = xdiv(xmul(p.lambda_v, p.block_size), p.sound_speed);
    const double rm = xmul(p.block_size, p.mass);
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < p.n_cells;
         c += gridDim.x * blockDim.x)
        b.block_raw[c] = assign_cell(p, b, c, sound_bound, rm);
}

// assign + smooth in one pass: each CTA assigns a tile of blocks plus a
// one-block halo into shared memory, then smooths the tile from there
// (WCSPH's level field, rts_block_levels expand = 0)
constexpr int kTX = 4, kTY = 8, kTZ = 32;
constexpr int kHX = kTX + 2, kHY = kTY + 2, kHZ = kTZ + 2;
constexpr int kHalo = kHX * kHY * kHZ;
constexpr int kHaloPer = (kHalo + 255) / 256;  // halo cells per thread (256 threads)

__global__ void __launch_bounds__(256) k_assign_smooth(const __grid_constant__ RtsParams p,
                                                       RtsBuffers b, int8_t *out) {
    if (fatal(b.ctr)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) b.ctr->stamps[1] = gtimer();  // grid rebuilt
    __shared__ int8_t s_reg[kHX * kHY * kHZ];
    const int nx = p.dims[0], ny = p.dims[1], nz = p.dims[2];
    const int tx = (nx + kTX - 1) / kTX, ty = (ny + kTY - 1) / kTY, tz = (nz + kTZ - 1) / kTZ;
    const double sound_bound = xdiv(xmul(p.lambda_v, p.block_size), p.sound_speed);
    const double rm = xmul(p.block_size, p.mass);
    for (int t = blockIdx.x; t < tx * ty * tz; t += gridDim.x) {
        const int bz = (t % tz) * kTZ, by = ((t / tz) % ty) * kTY, bx = (t / (tz * ty)) * kTX;
        // the halo's counts, then the occupied cells' maxima, all requested
        // before any is used (one dependent round trip each, not kHaloPer)
        int cell[kHaloPer], cnt[kHaloPer];
        double vm[kHaloPer], fm[kHaloPer];
#pragma unroll
        for (int u = 0; u < kHaloPer; ++u) {
            const int h = threadIdx.x + u * 256;
            const int hz = h % kHZ, hy = (h / kHZ) % kHY, hx = h / (kHZ * kHY);
            const int cx = bx + hx - 1, cy = by + hy - 1, cz = bz + hz - 1;
            const bool in = h < kHalo && cx >= 0 && cx < nx && cy >= 0 && cy < ny && cz >= 0 &&
                            cz < nz;
            cell[u] = in ? (cx * ny + cy) * nz + cz : -1;
            cnt[u] = in ? __ldg(b.cell_count + cell[u]) : 0;
        }
#pragma unroll
        for (int u = 0; u < kHaloPer; ++u) {
            vm[u] = cnt[u] > 0 ? __ldg(b.vmax + cell[u]) : 0.0;
            fm[u] = cnt[u] > 0 ? __ldg(b.fmax + cell[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kHaloPer; ++u) {
            const int h = threadIdx.x + u * 256;
            if (h >= kHalo) break;
            // outside the grid or empty: 0
            const int8_t r = cnt[u] > 0 ? assign_from(p, vm[u], fm[u], sound_bound, rm) : 0;
            const int hz = h % kHZ, hy = (h / kHZ) % kHY, hx = h / (kHZ * kHY);
            const bool interior = hx >= 1 && hx <= kTX && hy >= 1 && hy <= kTY && hz >= 1 &&
                                  hz <= kTZ;
            if (interior && cell[u] >= 0) b.block_raw[cell[u]] = r;
            s_reg[h] = r;
        }
        __syncthreads();
        for (int q = threadIdx.x; q < kTX * kTY * kTZ; q += blockDim.x) {
            const int iz = q % kTZ, iy = (q / kTZ) % kTY, ix = q / (kTZ * kTY);
            const int cx = bx + ix, cy = by + iy, cz = bz + iz;
            if (cx >= nx || cy >= ny || cz >= nz) continue;
            const int8_t f = s_reg[((ix + 1) * kHY + iy + 1) * kHZ + iz + 1];
            int8_t res = 0;
            if (f > 0) {
                if (p.pin_region) {
                    res = (int8_t)p.pin_region;
                } else {
                    int8_t m = kEmpty;
                    for (int dx = 0; dx < 3; ++dx)
                        for (int dy = 0; dy < 3; ++dy)
                            for (int dz = 0; dz < 3; ++dz) {
                                if (dx == 1 && dy == 1 && dz == 1) continue;
                                const int8_t v = s_reg[((ix + dx) * kHY + iy + dy) * kHZ + iz + dz];
                                if (v > 0 && v < m) m = v;
                            }
                    res = f < m ? f : m;
                }
            }
            out[(cx * ny + cy) * nz + cz] = res;
        }
        __syncthreads();
    }
}

// new = min(own, min over 26 occupied neighbours), empty stays 0
__global__ void k_smooth(const __grid_constant__ RtsParams p, RtsBuffers b, int8_t *out) {
    if (fatal(b.ctr)) return;
    const int nx = p.dims[0], ny = p.dims[1], nz = p.dims[2];
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < p.n_cells;
         c += gridDim.x * blockDim.x) {
        const int8_t f = b.block_raw[c];
        int8_t res = 0;
        if (f > 0) {
            if (p.pin_region) {
                res = (int8_t)p.pin_region;
            } else {
                const int cz = c % nz, cy = (c / nz) % ny, cx = c / (ny * nz);
                int8_t m = kEmpty;
                for (int ax = max(0, cx - 1); ax <= min(nx - 1, cx + 1); ++ax)
                    for (int ay = max(0, cy - 1); ay <= min(ny - 1, cy + 1); ++ay) {
                        const int base = (ax * ny + ay) * nz;
                        for (int az = max(0, cz - 1); az <= min(nz - 1, cz + 1); ++az) {
                            const int q = base + az;
                            if (q == c) continue;
                            const int8_t v = b.block_raw[q];
                            if (v > 0 && v < m) m = v;
                        }
                    }
                res = f < m ? f : m;
            }
        }
        out[c] = res;
    }
}

// separable Chebyshev dilation of the two masks {f==2 -> bit0, f==1 -> bit1}
__global__ void k_dilate_axis(const __grid_constant__ RtsParams p, const int8_t *field,
                              const uint8_t *in, uint8_t *out, int axis, int layers,
                              int from_field) {
    const int nx = p.dims[0], ny = p.dims[1], nz = p.dims[2];
    const int dim = p.dims[axis];
    const int stride = axis == 0 ? ny * nz : (axis == 1 ? nz : 1);
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < p.n_cells;
         c += gridDim.x * blockDim.x) {
        const int coord = axis == 0 ? c / (ny * nz) : (axis == 1 ? (c / nz) % ny : c % nz);
        uint8_t acc = 0;
        const int lo = max(0, coord - layers), hi = min(dim - 1, coord + layers);
        for (int q = lo; q <= hi; ++q) {
            const int cc = c + (q - coord) * stride;
            uint8_t v;
            if (from_field) {
                const int8_t f = field[cc];
                v = (uint8_t)((f == 2 ? 1 : 0) | (f == 1 ? 2 : 0));
            } else {
                v = in[cc];
            }
            acc |= v;
        }
        out[c] = acc;
    }
    (void)nx;
}

// regions.py:101-107: occupied blocks with a larger region inside a dilated
// mask drop to 2, then (taking precedence) to 1
__global__ void k_expand_apply(const __grid_constant__ RtsParams p, const int8_t *field,
                               const uint8_t *near, int8_t *out) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < p.n_cells;
         c += gridDim.x * blockDim.x) {
        const int8_t f = field[c];
        int8_t v = f;
        if (f > 2 && (near[c] & 1)) v = 2;
        if (f > 1 && (near[c] & 2)) v = 1;
        out[c] = v;
    }
}

// derive_observed (regions.py:110-125) for a caller-provided error mask
// (block_flag): occupied and (bordering a strictly smaller region, or
// bordering an error block without being one); -> block_tmp
__global__ void k_observed_mask(const __grid_constant__ RtsParams p, RtsBuffers b) {
    const int nx = p.dims[0], ny = p.dims[1], nz = p.dims[2];
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < p.n_cells;
         c += gridDim.x * blockDim.x) {
        const int8_t f = b.block_field[c];
        bool obs = false;
        if (f > 0) {
            const int cz = c % nz, cy = (c / nz) % ny, cx = c / (ny * nz);
            int8_t m = kEmpty;
            bool near_err = false;
            for (int ax = max(0, cx - 1); ax <= min(nx - 1, cx + 1); ++ax)
                for (int ay = max(0, cy - 1); ay <= min(ny - 1, cy + 1); ++ay) {
                    const int base = (ax * ny + ay) * nz;
                    for (int az = max(0, cz - 1); az <= min(nz - 1, cz + 1); ++az) {
                        const int q = base + az;
                        if (q == c) continue;
                        const int8_t v = b.block_field[q];
                        if (v > 0 && v < m) m = v;
                        near_err = near_err || b.block_flag[q];
                    }
                }
            obs = (m < f) || (near_err && !b.block_flag[c]);
        }
        b.block_tmp[c] = obs;
    }
}

// neighbor_min (grid.py:33-45) of an int8 field in block_raw, out-of-grid
// cells = pad; -> block_field
__global__ void k_neighbor_min(const __grid_constant__ RtsParams p, RtsBuffers b, int pad) {
    const int nx = p.dims[0], ny = p.dims[1], nz = p.dims[2];
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < p.n_cells;
         c += gridDim.x * blockDim.x) {
        const int cz = c % nz, cy = (c / nz) % ny, cx = c / (ny * nz);
        int m = pad;
        for (int ax = cx - 1; ax <= cx + 1; ++ax)
            for (int ay = cy - 1; ay <= cy + 1; ++ay)
                for (int az = cz - 1; az <= cz + 1; ++az) {
                    if (ax == cx && ay == cy && az == cz) continue;
                    const bool in = ax >= 0 && ax < nx && ay >= 0 && ay < ny && az >= 0 && az < nz;
                    const int v = in ? (int)b.block_raw[(ax * ny + ay) * nz + az] : pad;
                    m = v < m ? v : m;
                }
        b.block_field[c] = (int8_t)m;
    }
}

}  // namespace

extern "C" int rts_block_levels(const RtsParams *p, const RtsBuffers *b, int expand,
                                void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int blocks = rts_blocks(p->n_cells, kThreads);
    if (expand == 2) {  // assign only (required levels, pcisph.py:726-740)
        rts_note_launch(), k_assign<<<blocks, kThreads, 0, s>>>(*p, *b);
        RTS_LAUNCH_CHECK();
        return 0;
    }
    const long long tiles = (long long)((p->dims[0] + kTX - 1) / kTX) *
                            ((p->dims[1] + kTY - 1) / kTY) * ((p->dims[2] + kTZ - 1) / kTZ);
    const int tb = (int)(tiles < 148 * 8 ? tiles : 148 * 8);
    if (!expand || p->pin_region) {  // assign + smooth -> block_field
        rts_note_launch(), k_assign_smooth<<<tb, 256, 0, s>>>(*p, *b, b->block_field);
        RTS_LAUNCH_CHECK();
        return 0;
    }
    // assign + smooth into block_tmp, then the expansion into block_field
    rts_note_launch(), k_assign_smooth<<<tb, 256, 0, s>>>(*p, *b, b->block_tmp);
    RTS_LAUNCH_CHECK();
    uint8_t *m0 = b->block_flag;
    uint8_t *m1 = reinterpret_cast<uint8_t *>(b->block_field);  // scratch until final write
    rts_note_launch(), k_dilate_axis<<<blocks, kThreads, 0, s>>>(*p, b->block_tmp, nullptr, m0, 2, 4, 1);
    rts_note_launch(), k_dilate_axis<<<blocks, kThreads, 0, s>>>(*p, nullptr, m0, m1, 1, 4, 0);
    rts_note_launch(), k_dilate_axis<<<blocks, kThreads, 0, s>>>(*p, nullptr, m1, m0, 0, 4, 0);
    rts_note_launch(), k_expand_apply<<<blocks, kThreads, 0, s>>>(*p, b->block_tmp, m0, b->block_field);
    RTS_LAUNCH_CHECK();
    return 0;
}

// The regions.py functions on caller-provided fields (the public API of the
// reference: smooth_regions, expand_fast_regions, derive_observed).
//   op 0: smooth   block_raw -> block_field
//   op 1: expand   block_tmp -> block_field, `arg` layers (scratch: block_flag)
//   op 2: observed block_field + error mask block_flag -> block_tmp
//   op 3: neighbour minimum of block_raw (out-of-grid = arg) -> block_field
extern "C" int rts_region_op(const RtsParams *p, const RtsBuffers *b, int op, int arg,
                             void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int blocks = rts_blocks(p->n_cells, kThreads);
    if (op == 0) {
        rts_note_launch(), k_smooth<<<blocks, kThreads, 0, s>>>(*p, *b, b->block_field);
    } else if (op == 1) {
        uint8_t *m0 = b->block_flag;
        uint8_t *m1 = reinterpret_cast<uint8_t *>(b->block_raw);  // scratch
        rts_note_launch(), k_dilate_axis<<<blocks, kThreads, 0, s>>>(*p, b->block_tmp, nullptr, m0, 2, arg, 1);
        rts_note_launch(), k_dilate_axis<<<blocks, kThreads, 0, s>>>(*p, nullptr, m0, m1, 1, arg, 0);
        rts_note_launch(), k_dilate_axis<<<blocks, kThreads, 0, s>>>(*p, nullptr, m1, m0, 0, arg, 0);
        rts_note_launch(), k_expand_apply<<<blocks, kThreads, 0, s>>>(*p, b->block_tmp, m0, b->block_field);
    } else if (op == 2) {
        rts_note_launch(), k_observed_mask<<<blocks, kThreads, 0, s>>>(*p, *b);
    } else if (op == 3) {
        rts_note_launch(), k_neighbor_min<<<blocks, kThreads, 0, s>>>(*p, *b, arg);
    } else {
        return (int)cudaErrorInvalidValue;
    }
    RTS_LAUNCH_CHECK();
    return 0;
}
