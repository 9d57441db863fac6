/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the RTS-SPH hot path.
 *
 * Plain-C (fp64, OpenMP) restatement of the compiled particle loops of the
 * reference package `rts_sph` (arXiv 2009.14514).  This file is the checker
 * the B200 kernels are compared against; it is never linked into, called by
 * or shipped with the product library (paper_2009_14514_b200/csrc).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm load it.
 *
 * Arithmetic is written operation-for-operation in the reference's order
 * and the file is built with -ffp-contract=off, so every result is bit-for-
 * bit the value the reference's LLVM-compiled loops produce (pinned by
 * tests/test_oracle_golden.py against fixtures generated from the reference
 * itself by tests/golden/make_golden.py).
 *
 * Each function cites the reference loop it restates (path:line into
 * /root/reference/pkg/src/rts_sph).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define EXPORT __attribute__((visibility("default")))

static inline int64_t clamp_cell(int64_t c, int64_t n) {
    if (c < 0) return 0;
    if (c >= n) return n - 1;
    return c;
}

/* Cell of a point from C-style truncation, as the search loops do
 * (grid.py:116-131): int() truncates toward zero, then clamp. */
static inline int64_t trunc_cell(double x, double o, double inv, int64_t n) {
    return clamp_cell((int64_t)((x - o) * inv), n);
}

EXPORT int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

EXPORT void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* grid.py:70-85 -- stable counting sort of cell ids into CSR (starts, order). */
EXPORT void oracle_counting_sort(const int64_t *cell_ids, int64_t n, int64_t n_cells,
                                 int64_t *starts, int64_t *order) {
    memset(starts, 0, sizeof(int64_t) * (size_t)(n_cells + 1));
    for (int64_t k = 0; k < n; ++k) starts[cell_ids[k] + 1] += 1;
    for (int64_t c = 0; c < n_cells; ++c) starts[c + 1] += starts[c];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_cells > 0 ? n_cells : 1));
    memcpy(fill, starts, sizeof(int64_t) * (size_t)n_cells);
    for (int64_t k = 0; k < n; ++k) {
        int64_t c = cell_ids[k];
        order[fill[c]++] = k;
    }
    free(fill);
}

/* grid.py:88-152 -- per refresh particle, scan (2L+1)^3 blocks around the
 * particle's current block and store every j with r^2 < h^2 (self included)
 * into row i of the fixed-width table.  Returns entries lost to overflow. */
EXPORT int64_t oracle_search_neighbors(const double *pos, const int64_t *starts,
                                       const int64_t *order, int64_t nx, int64_t ny,
                                       int64_t nz, const double *origin, double inv_r,
                                       double h2, const int64_t *refresh, int64_t n_refresh,
                                       const int64_t *layers, int64_t *nbr, int64_t width,
                                       int64_t *cnt) {
    int64_t overflow = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : overflow)
    for (int64_t t = 0; t < n_refresh; ++t) {
        const int64_t i = refresh[t];
        const int64_t lay = layers[t];
        const double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
        const int64_t cx = trunc_cell(xi, origin[0], inv_r, nx);
        const int64_t cy = trunc_cell(yi, origin[1], inv_r, ny);
        const int64_t cz = trunc_cell(zi, origin[2], inv_r, nz);
        int64_t n = 0, lost = 0;
        int64_t *row = nbr + i * width;
        const int64_t ax0 = cx - lay > 0 ? cx - lay : 0, ax1 = cx + lay + 1 < nx ? cx + lay + 1 : nx;
        const int64_t ay0 = cy - lay > 0 ? cy - lay : 0, ay1 = cy + lay + 1 < ny ? cy + lay + 1 : ny;
        const int64_t az0 = cz - lay > 0 ? cz - lay : 0, az1 = cz + lay + 1 < nz ? cz + lay + 1 : nz;
        for (int64_t ax = ax0; ax < ax1; ++ax)
            for (int64_t ay = ay0; ay < ay1; ++ay) {
                const int64_t base = (ax * ny + ay) * nz;
                for (int64_t az = az0; az < az1; ++az) {
                    const int64_t c = base + az;
                    for (int64_t k = starts[c]; k < starts[c + 1]; ++k) {
                        const int64_t j = order[k];
                        const double dx = xi - pos[3 * j];
                        const double dy = yi - pos[3 * j + 1];
                        const double dz = zi - pos[3 * j + 2];
                        const double r2 = dx * dx + dy * dy + dz * dz;
                        if (r2 < h2) {
                            if (n < width) row[n++] = j;
                            else ++lost;
                        }
                    }
                }
            }
        cnt[i] = n;
        overflow += lost;
    }
    return overflow;
}

/* grid.py:155-162 -- per-cell running maximum (out pre-zeroed by caller). */
EXPORT void oracle_reduce_max(const double *values, const int64_t *cell_ids, int64_t n,
                              double *out) {
    for (int64_t k = 0; k < n; ++k) {
        const double v = values[k];
        if (v > out[cell_ids[k]]) out[cell_ids[k]] = v;
    }
}

/* grid.py:165-212 -- count true neighbours missing from freshly built tables,
 * scanning one layer of an exhaustive grid. */
EXPORT int64_t oracle_count_missing(const double *pos, const int64_t *starts, const int64_t *order,
                                    int64_t nx, int64_t ny, int64_t nz, const double *origin,
                                    double inv_r, double h2, const int64_t *refresh,
                                    int64_t n_refresh, const int64_t *nbr, int64_t width,
                                    const int64_t *cnt) {
    int64_t missing = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : missing)
    for (int64_t t = 0; t < n_refresh; ++t) {
        const int64_t i = refresh[t];
        const double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
        const int64_t cx = trunc_cell(xi, origin[0], inv_r, nx);
        const int64_t cy = trunc_cell(yi, origin[1], inv_r, ny);
        const int64_t cz = trunc_cell(zi, origin[2], inv_r, nz);
        const int64_t *row = nbr + i * width;
        int64_t lost = 0;
        for (int64_t ax = (cx - 1 > 0 ? cx - 1 : 0); ax < (cx + 2 < nx ? cx + 2 : nx); ++ax)
            for (int64_t ay = (cy - 1 > 0 ? cy - 1 : 0); ay < (cy + 2 < ny ? cy + 2 : ny); ++ay) {
                const int64_t base = (ax * ny + ay) * nz;
                for (int64_t az = (cz - 1 > 0 ? cz - 1 : 0); az < (cz + 2 < nz ? cz + 2 : nz); ++az) {
                    const int64_t c = base + az;
                    for (int64_t k = starts[c]; k < starts[c + 1]; ++k) {
                        const int64_t j = order[k];
                        const double dx = xi - pos[3 * j];
                        const double dy = yi - pos[3 * j + 1];
                        const double dz = zi - pos[3 * j + 2];
                        if (dx * dx + dy * dy + dz * dz < h2) {
                            int found = 0;
                            for (int64_t q = 0; q < cnt[i]; ++q)
                                if (row[q] == j) { found = 1; break; }
                            if (!found) ++lost;
                        }
                    }
                }
            }
        missing += lost;
    }
    return missing;
}

/* kernels.py:23-55 -- scalar kernel helpers, reference operation order. */
static inline double poly6(double r2, double h2, double c) {
    const double d = h2 - r2;
    if (d <= 0.0) return 0.0;
    return c * d * d * d;
}
static inline double spiky_scale(double r, double h, double c) {
    if (r <= 0.0 || r >= h) return 0.0;
    const double d = h - r;
    return c * d * d / r;
}
static inline double visc_lap(double r, double h, double c) {
    const double d = h - r;
    if (d <= 0.0) return 0.0;
    return c * d;
}

/* wcsph.py:45-60 -- density sum and clamped Tait pressure for idx.  The
 * seventh power is exponentiation by squaring, (x*x^2)*x^4, which is what the
 * reference's compiled `ratio**7` evaluates to (verified bit-for-bit). */
EXPORT void oracle_density_pressure(const double *pos, const int64_t *nbr, int64_t width,
                                    const int64_t *cnt, const int64_t *idx, int64_t n_idx,
                                    double mass, double h2, double c_poly6, double b_stiff,
                                    double rho0, double *rho, double *pres) {
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n_idx; ++t) {
        const int64_t i = idx[t];
        const int64_t *row = nbr + i * width;
        double acc = 0.0;
        for (int64_t k = 0; k < cnt[i]; ++k) {
            const int64_t j = row[k];
            const double dx = pos[3 * i] - pos[3 * j];
            const double dy = pos[3 * i + 1] - pos[3 * j + 1];
            const double dz = pos[3 * i + 2] - pos[3 * j + 2];
            acc += poly6(dx * dx + dy * dy + dz * dz, h2, c_poly6);
        }
        const double r = mass * acc;
        rho[i] = r;
        const double x = r / rho0;
        const double x2 = x * x;
        const double x4 = x2 * x2;
        const double p = b_stiff * ((x * x2) * x4 - 1.0);
        pres[i] = p > 0.0 ? p : 0.0;
    }
}

/* wcsph.py:63-105 -- symmetric pressure + laminar viscosity over fluid
 * neighbours, mirrored wall pressure for boundary neighbours, plus m*g. */
EXPORT void oracle_forces(const double *pos, const double *vel, const int64_t *nbr, int64_t width,
                          const int64_t *cnt, const int64_t *idx, int64_t n_idx, double mass,
                          double h, double c_spiky, double c_visc, double mu, double rho0,
                          int64_t n_fluid, const double *rho, const double *pres,
                          const double *grav, double *force) {
    const double m2 = mass * mass;
    const double inv_rho0_sq = 1.0 / (rho0 * rho0);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n_idx; ++t) {
        const int64_t i = idx[t];
        const int64_t *row = nbr + i * width;
        const double rho_i = rho[i];
        const double p_i = pres[i];
        const double term_i = p_i / (rho_i * rho_i);
        double fx = 0.0, fy = 0.0, fz = 0.0;
        for (int64_t k = 0; k < cnt[i]; ++k) {
            const int64_t j = row[k];
            if (j == i) continue;
            const double dx = pos[3 * i] - pos[3 * j];
            const double dy = pos[3 * i + 1] - pos[3 * j + 1];
            const double dz = pos[3 * i + 2] - pos[3 * j + 2];
            const double r = sqrt(dx * dx + dy * dy + dz * dz);
            if (r >= h) continue;
            if (j < n_fluid) {
                const double rho_j = rho[j];
                const double term = term_i + pres[j] / (rho_j * rho_j);
                const double s = m2 * term * spiky_scale(r, h, c_spiky);
                fx -= s * dx;
                fy -= s * dy;
                fz -= s * dz;
                const double lap = mu * m2 * visc_lap(r, h, c_visc) / (rho_i * rho_j);
                fx += lap * (vel[3 * j] - vel[3 * i]);
                fy += lap * (vel[3 * j + 1] - vel[3 * i + 1]);
                fz += lap * (vel[3 * j + 2] - vel[3 * i + 2]);
            } else {
                const double term = term_i + p_i * inv_rho0_sq;
                const double s = m2 * term * spiky_scale(r, h, c_spiky);
                fx -= s * dx;
                fy -= s * dy;
                fz -= s * dz;
            }
        }
        force[3 * i] = fx + mass * grav[0];
        force[3 * i + 1] = fy + mass * grav[1];
        force[3 * i + 2] = fz + mass * grav[2];
    }
}

/* pcisph.py:174-199 -- viscosity (1/rho0^2 form) + m*g for idx. */
EXPORT void oracle_ext_forces(const double *pos, const double *vel, const int64_t *nbr,
                              int64_t width, const int64_t *cnt, const int64_t *idx,
                              int64_t n_idx, double mass, double h, double c_visc, double mu,
                              double rho0, int64_t n_fluid, const double *grav, double *out) {
    const double m2 = mass * mass;
    const double inv_rho0_sq = 1.0 / (rho0 * rho0);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n_idx; ++t) {
        const int64_t i = idx[t];
        const int64_t *row = nbr + i * width;
        double fx = 0.0, fy = 0.0, fz = 0.0;
        for (int64_t k = 0; k < cnt[i]; ++k) {
            const int64_t j = row[k];
            if (j >= n_fluid || j == i) continue;
            const double dx = pos[3 * i] - pos[3 * j];
            const double dy = pos[3 * i + 1] - pos[3 * j + 1];
            const double dz = pos[3 * i + 2] - pos[3 * j + 2];
            const double r = sqrt(dx * dx + dy * dy + dz * dz);
            if (r >= h) continue;
            const double lap = mu * m2 * visc_lap(r, h, c_visc) * inv_rho0_sq;
            fx += lap * (vel[3 * j] - vel[3 * i]);
            fy += lap * (vel[3 * j + 1] - vel[3 * i + 1]);
            fz += lap * (vel[3 * j + 2] - vel[3 * i + 2]);
        }
        out[3 * i] = fx + mass * grav[0];
        out[3 * i + 1] = fy + mass * grav[1];
        out[3 * i + 2] = fz + mass * grav[2];
    }
}

/* pcisph.py:202-213 -- predicted velocity and position for all fluid. */
EXPORT void oracle_predict_motion(const double *pos, const double *vel, const double *f_ext,
                                  const double *f_p, int64_t n_fluid, double dt, double inv_mass,
                                  double *xstar, double *vstar) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_fluid; ++i) {
        for (int a = 0; a < 3; ++a) {
            const double v = vel[3 * i + a] + dt * inv_mass * (f_ext[3 * i + a] + f_p[3 * i + a]);
            vstar[3 * i + a] = v;
        }
        for (int a = 0; a < 3; ++a) xstar[3 * i + a] = pos[3 * i + a] + dt * vstar[3 * i + a];
    }
}

/* pcisph.py:216-235 -- predicted density over cached lists (fluid
 * neighbours at x*, boundary at pos) and the clamped compression error. */
EXPORT void oracle_predict_density(const double *xstar, const double *pos, const int64_t *nbr,
                                   int64_t width, const int64_t *cnt, const int64_t *idx,
                                   int64_t n_idx, double mass, double h2, double c_poly6,
                                   double rho0, int64_t n_fluid, double *rho_star, double *err) {
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n_idx; ++t) {
        const int64_t i = idx[t];
        const int64_t *row = nbr + i * width;
        double acc = 0.0;
        for (int64_t k = 0; k < cnt[i]; ++k) {
            const int64_t j = row[k];
            const double *pj = j < n_fluid ? xstar + 3 * j : pos + 3 * j;
            const double dx = xstar[3 * i] - pj[0];
            const double dy = xstar[3 * i + 1] - pj[1];
            const double dz = xstar[3 * i + 2] - pj[2];
            acc += poly6(dx * dx + dy * dy + dz * dz, h2, c_poly6);
        }
        const double r = mass * acc;
        rho_star[i] = r;
        const double diff = r - rho0;
        err[i] = diff > 0.0 ? diff / rho0 : 0.0;
    }
}

/* pcisph.py:238-271 -- pressure forces at predicted positions. */
EXPORT void oracle_pressure_forces(const double *xstar, const double *pos, const int64_t *nbr,
                                   int64_t width, const int64_t *cnt, const int64_t *idx,
                                   int64_t n_idx, double mass, double h, double c_spiky,
                                   double rho0, int64_t n_fluid, const double *p, double *out) {
    const double m2 = mass * mass;
    const double inv_rho0_sq = 1.0 / (rho0 * rho0);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n_idx; ++t) {
        const int64_t i = idx[t];
        const int64_t *row = nbr + i * width;
        const double term_i = p[i] * inv_rho0_sq;
        double fx = 0.0, fy = 0.0, fz = 0.0;
        for (int64_t k = 0; k < cnt[i]; ++k) {
            const int64_t j = row[k];
            if (j == i) continue;
            double dx, dy, dz, term;
            if (j < n_fluid) {
                dx = xstar[3 * i] - xstar[3 * j];
                dy = xstar[3 * i + 1] - xstar[3 * j + 1];
                dz = xstar[3 * i + 2] - xstar[3 * j + 2];
                term = term_i + p[j] * inv_rho0_sq;
            } else {
                dx = xstar[3 * i] - pos[3 * j];
                dy = xstar[3 * i + 1] - pos[3 * j + 1];
                dz = xstar[3 * i + 2] - pos[3 * j + 2];
                term = term_i + term_i;
            }
            const double r = sqrt(dx * dx + dy * dy + dz * dz);
            if (r <= 0.0 || r >= h) continue;
            const double s = m2 * term * spiky_scale(r, h, c_spiky);
            fx -= s * dx;
            fy -= s * dy;
            fz -= s * dz;
        }
        out[3 * i] = fx;
        out[3 * i + 1] = fy;
        out[3 * i + 2] = fz;
    }
}

/* numpy's pairwise summation (the algorithm behind ndarray.sum/mean for
 * contiguous float64), restated so the oracle's average-error figure
 * (pcisph.py:421-430) matches the reference bit for bit. */
static double pairwise_sum(const double *a, int64_t n) {
    if (n < 8) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += a[i];
        return s;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) s += a[i];
        return s;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
}

EXPORT double oracle_pairwise_sum(const double *a, int64_t n) { return pairwise_sum(a, n); }
