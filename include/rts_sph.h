/*
 * rts_sph.h -- C ABI of librtssph.so, the B200 (sm_100a) kernels behind the
 * RTS-SPH drop-in (arXiv 2009.14514; reference package rts_sph at
 * /root/reference/pkg/src/rts_sph).
 *
 * The reference has no FFI: its operator seam is a set of Numba @njit loops
 * called from Python with caller-owned arrays.  Each entry point below
 * replaces one of those loops (or one numpy pass around them) and cites it.
 *
 * Conventions
 *   - All pointers are device pointers owned by the caller (the Python host
 *     package allocates them with torch); the library never allocates or
 *     frees device memory.
 *   - `stream` is a cudaStream_t passed as void*; every entry point only
 *     enqueues work on it (asynchronous, no host synchronisation).
 *   - Return value: 0 on success, otherwise a cudaError_t code from the
 *     launch.  Data errors (escaped particles, overflow, non-finite
 *     density, iteration cap) never return non-zero: kernels record them in
 *     RtsCounters.err_flags, which the host reads once per step / minor step
 *     and raises as NumericalError with the reference's message.
 *   - Once a fatal flag is set, every later kernel of the step returns
 *     immediately, so the state is left as it was when the step began, as
 *     with the reference's exceptions.
 *   - Particle state is fp32 (float3 rows); geometry decisions (block keys,
 *     r^2 < h^2 membership, region levels) and the density / EOS sums are
 *     evaluated in fp64 with un-fused operations in the reference's order.
 */
#ifndef RTS_SPH_H
#define RTS_SPH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RTS_ABI_VERSION 28

/* err_flags bits */
#define RTS_ERR_ESCAPED   0x1u  /* fluid left the padded grid or non-finite (grid.py:268-273) */
#define RTS_ERR_OVERFLOW  0x2u  /* > width true neighbours (grid.py:327-331) */
#define RTS_ERR_NONFINITE 0x4u  /* non-finite density (wcsph.py:286-287, pcisph.py:680-681) */
#define RTS_ERR_ITERCAP   0x8u  /* pressure solve hit the cap (pcisph.py:711-715) */
#define RTS_ERR_CHECK     0x10u /* checked builds (-DRTS_CHECKED=1): a device index was out of
                                 * range; RtsCounters.check_site names the first site */
#define RTS_ERR_FATAL     0x1Fu

/* Scalar constants of one solver, fp64 values computed by the Python host
 * with the reference's own expressions (scene.py, kernels.py:58-80,
 * wcsph.py:143-150, pcisph.py:308-321). */
typedef struct RtsParams {
    double origin[3];      /* grid.py:225-229 */
    double grid_hi[3];     /* origin + dims*block, domain-check bound (grid.py:266) */
    double block_size;
    double inv_block;
    double h, h2, c_poly6, c_spiky, c_visc;
    double mass, inv_mass, rho0, b_stiff, mu;
    double clamp_lo[3], clamp_hi[3];   /* wcsph.py:171-172 */
    double gravity[3];
    double dt;             /* step length of this call */
    double dt_base, lambda_v, lambda_f, sound_speed, alpha;
    double betas[8];       /* scene.py:130-139, index = region id */
    double eta_max, eta_avg, rho_T, delta;   /* PCISPH (scene.py:91-93, pcisph.py:359-361) */
    int32_t dims[3];
    int32_t n_cells;
    int32_t n_fluid;
    int32_t n_bound;
    int32_t n_bcells;      /* distinct cells holding boundary particles */
    int32_t width;         /* neighbour table width (wcsph.py:35) */
    int32_t n_max;         /* largest region id for assign_regions */
    int32_t use_sound;     /* WCSPH uses the acoustic criterion */
    int32_t pin_region;    /* 0 = off, else force every occupied block */
    int32_t apply_correction;
    int32_t rts;           /* 1 = regional mode, 0 = synchronous baseline */
    int32_t n_sms;         /* grid sizing for persistent kernels */
    int32_t n_regions;     /* region ids 1..n_regions (pcisph.py:294) */
    int32_t n_global;      /* fluid count of the whole scene (x-slab ranks); 0 = n_fluid */
    int32_t nbr_stride;    /* column stride of the neighbour table: entry q of particle i
                            * is nbr[q * nbr_stride + i] (column-major, coalesced reads) */
    int32_t n_ghost;       /* ghost rows among the n_fluid (x-slab ranks; 0 otherwise) */
} RtsParams;

/* Device-side counters; copied to the host once per step. */
typedef struct RtsCounters {
    uint32_t err_flags;
    int32_t  n_escaped;        /* count of bad fluid rows */
    int32_t  first_escaped;    /* lowest bad index (INT32_MAX if none) */
    int32_t  n_compute;        /* active particles this step */
    int64_t  overflow;         /* neighbour entries beyond width */
    int32_t  n_sorted;         /* fluid + active boundary in the CSR */
    int32_t  n_pred;           /* PCISPH: |pred set| of the current iteration */
    int32_t  n_force;          /* PCISPH: |force set| of the current iteration */
    int32_t  n_list;           /* generic compacted list length */
    uint64_t fmax_bits;        /* max |F| over fluid (baseline CFL), double bits */
    double   sum_rho;          /* PCISPH: sum of rho* over fluid */
    double   max_err;          /* PCISPH: max err over fluid */
    int32_t  any_se;           /* PCISPH: any particle in S_e */
    int32_t  lists_all;        /* PCISPH: this iteration's pred = force = all fluid (no lists) */
    int64_t  missing;          /* neighbour audit: true neighbours absent from tables */
    uint32_t blocks_done;      /* last-block-done counter of the S_e reduction */
    int32_t  check_site;       /* checked builds: first failing RTS_CHECK site (0 = none) */
    int64_t  stamps[4];        /* RTS-WCSPH step graph: %globaltimer (ns) at the start, end of
                                * the grid rebuild, start of the density pass, end */
    float    disp_cur;         /* PCISPH: max |dx| of one coordinate of any fluid particle in
                                * the current minor step's integration (>= 0 float bits) */
    float    disp_total;       /* PCISPH: sum of disp_cur over the completed minor steps of
                                * this major: bound on any coordinate's displacement since
                                * the rebuild (the partial refreshes cull by it) */
    int32_t  soa_fresh;        /* PCISPH: the x / y / z candidate copies match cpos (set by
                                * the gather at a major start, cleared by the integrator,
                                * which keeps only cpos current) */
    int32_t  reserved1;
} RtsCounters;

/* Per-minor-step record written by the device loop control (StepStats,
 * stats.py:9-40 / pcisph.py:591-610). */
typedef struct RtsMinorStats {
    int32_t  iterations;
    int32_t  n_refresh;
    int32_t  early;
    int32_t  riters[5];
    int64_t  corrected;
    int64_t  forced;       /* sum of |force set| over the iterations */
    double   max_err;
    double   avg_err;
    int64_t  t_begin, t_refreshed, t_looped, t_end;  /* %globaltimer ns */
} RtsMinorStats;

#define RTS_MAX_MINOR 8
#define RTS_MAX_ROWS 8

/* Device-resident state of the scheduled correction loop
 * (_correct_scheduled, pcisph.py:612-716; _correct_all, pcisph.py:439-468).
 * The k_control kernel owns every decision; iteration kernels only read
 * row_mask / motion_all / snap_op / done. */
typedef struct RtsControl {
    int32_t it, g_count, local_active, local_banned, local_run, early, done, failed;
    int32_t motion_all;    /* next motion pass covers all fluid */
    int32_t row_mask;      /* next iteration's scheduled regions (bit n), 0 = local pass */
    int32_t snap_op;       /* after control: 0 none, 1 snapshot p/f_p, 2 revert */
    int32_t minor;
    int32_t stop_major;    /* early termination or failure: later minors are skipped */
    int32_t local_entered, local_reverted;
    int32_t fail_kind;     /* 1 non-finite, 2 RTS cap, 3 sync cap */
    int32_t fail_g;
    int32_t stamp;         /* S_e generation: cells stamped with it hold S_e particles */
    int32_t prev_force;    /* |force set| of the previous iteration (motion list length) */
    int32_t n_rows[RTS_MAX_MINOR];
    int32_t row_masks[RTS_MAX_MINOR][RTS_MAX_ROWS];
    int32_t row_counts[RTS_MAX_MINOR][RTS_MAX_ROWS];  /* region multiplicities, 4 bits each */
    int32_t riters[5];
    int32_t skipped;       /* current minor skipped (stop_major) */
    int64_t corrected;
    int64_t forced;
    double  last_max_err, last_avg_err;
    double  fail_err;
    RtsMinorStats stats[RTS_MAX_MINOR];
} RtsControl;

/* Buffers: every pointer is caller-owned device memory. Sizes in comments,
 * Nf = n_fluid, Nb = n_bound, Nc = n_cells, Bc = n_bcells. */
typedef struct RtsBuffers {
    /* canonical particle state (index = reference particle index) */
    float   *pos;          /* (Nf+Nb, 3) */
    float   *vel;          /* (Nf, 3) */
    float   *acc;          /* (Nf, 3)  WCSPH */
    float   *acc_prev;     /* (Nf, 3)  WCSPH */
    float   *force;        /* (Nf, 3)  WCSPH force / PCISPH f_ext */
    float   *f_p;          /* (Nf, 3)  PCISPH pressure force */
    float   *rho;          /* (Nf)     WCSPH rho / PCISPH rho_star */
    float   *pres;         /* (Nf)     WCSPH pres / PCISPH p */
    double  *err;          /* (Nf)     PCISPH err (fp64: S_e threshold decisions) */
    float   *xstar;        /* (Nf, 3)  PCISPH x* */
    double  *dt_since;     /* (Nf) */
    double  *dt_corr;      /* (Nf) */
    int32_t *validity;     /* (Nf) */
    int8_t  *region;       /* (Nf) */
    uint8_t *compute;      /* (Nf) */
    uint8_t *in_se;        /* (Nf) */
    uint8_t *in_sob;       /* (Nf) */
    /* block grid */
    int32_t *fluid_cells;  /* (Nf) */
    int32_t *cell_count;   /* (Nc) fluid count per block */
    int32_t *cell_bcount;  /* (Nc) active boundary count per block (0 off boundary blocks) */
    int32_t *starts;       /* (Nc+1) CSR starts (grid.py:291) */
    int32_t *order;        /* (Nf+Nb) CSR members (grid.py:293) */
    int32_t *fill;         /* (Nc) scratch */
    int32_t *scan_tmp;     /* (>= 2*ceil(Nc/1024)+64) scratch */
    int32_t *bcell_ids;    /* (Bc) sorted block ids holding boundary particles */
    int32_t *bcell_start;  /* (Bc+1) CSR into bidx */
    int32_t *bidx;         /* (Nb) boundary particle indices (Nf + b), grouped by block */
    int32_t *bcell_of;     /* (Nb) index into bcell_ids of the block of bidx[q] */
    uint8_t *bcell_active; /* (Bc) */
    /* block fields */
    double  *vmax;         /* (Nc) per-block max |v| (grid.py:347) */
    double  *fmax;         /* (Nc) per-block max |F| */
    int8_t  *block_raw;    /* (Nc) assign_regions output */
    int8_t  *block_field;  /* (Nc) smoothed (and expanded) region field */
    int8_t  *block_tmp;    /* (Nc) scratch */
    uint8_t *block_flag;   /* (Nc) scratch mask (S_e blocks / observed) */
    /* sorted candidate copies, slot k of the CSR */
    float   *cpos;         /* (Nf+Nb, 4)  x y z p   (p = -1 marks a boundary slot) */
    float   *cvel;         /* (Nf+Nb, 4)  vx vy vz rho */
    double  *cterm;        /* (Nf+Nb, 4)  WCSPH: 32-byte rows {fp64 p/rho^2, fp64 1/rho, fp32 v}
                            * of the slot's particle (this step's density pass for active
                            * slots): one 256-bit gather per force pair */
    double  *cwall;        /* (Nf+Nb)     WCSPH: fp64 p/rho^2 + p/rho0^2 (wall pair term) */
    float   *cx, *cy, *cz; /* (Nf+Nb+4 each, 16-byte aligned) the candidate positions of cpos
                            * as separate x / y / z arrays: the neighbour searches load four
                            * candidates per 128-bit access and test them in packed fp32x2 */
    int32_t *active;       /* (Nf) compacted CSR slots of active fluid particles */
    int32_t *list2;        /* (Nf) second compacted list */
    int32_t *list3;        /* (Nf) PCISPH: force list of the previous iteration (motion
                            * input; written by the pressure-force pass, so k_sets may
                            * rebuild list2 concurrently with k_motion) */
    /* PCISPH neighbour tables */
    int32_t *nbr;          /* (width, nbr_stride) column-major neighbour particle indices
                            * (grid.py:146-149 rows, transposed) */
    int32_t *cnt;          /* (Nf) */
    double  *xs;           /* (Nf+Nb, 4) fp64 rows {x*, p}: the pressure solve's state
                            * (pres is p's fp32 mirror); wall rows {pos, -1} */
    uint8_t *pflag;        /* (Nf) per-iteration set bits (1 = force set) */
    double  *partial;      /* (>= 4096) deterministic reduction partials */
    double  *snap_p;       /* (Nf)    local-phase snapshot of the fp64 p (xs rows) */
    float   *snap_fp;      /* (Nf, 3) local-phase snapshot of f_p */
    int32_t *slot_of;      /* (Nf) CSR slot of each fluid particle (inverse of order) */
    RtsControl *ctl;       /* correction-loop control block */
    int32_t *se_stamp;     /* (Nc) S_e generation that last marked the block */
    int32_t *near_stamp;   /* (Nc) S_e generation that last marked a 26-neighbour */
    uint8_t *ghost;        /* (Nf) 1 = ghost row owned by another rank (or NULL) */
    int32_t *sort_key;     /* (Nf) global ids of the fluid rows: within-block CSR order by key
                            * instead of by row (x-slab ranks; NULL = by row) */
    RtsCounters *ctr;
} RtsBuffers;

/* ---- library ---------------------------------------------------------- */
int rts_abi_version(void);
/* Query the current device; returns its SM count or a negative cudaError. */
int rts_device_sms(void);
/* Number of librtssph kernels launched (or captured into graphs) by this
 * process so far. */
long long rts_launch_count(void);
/* Zero-filled cudaMemsetAsync helper so hosts need not link cudart. */
int rts_memset(void *dst, int value, int64_t bytes, void *stream);

/* Reset the counters block (err_flags = 0, first_escaped = INT32_MAX ...). */
int rts_counters_reset(const RtsBuffers *b, void *stream);
/* stamps[slot] = %globaltimer (one-thread kernel; phase timing inside graphs). */
int rts_stamp(const RtsBuffers *b, int slot, void *stream);

/* ---- block grid (grid.py) -------------------------------------------- */
/* One-time static binning of the boundary shell: bcell_of, and
 * bcell_ids/bcell_start/bidx (host computes the sort; see grid.py:279-290). */
/* Fluid block keys, domain check, occupancy counts; per-block max |v|, |F|
 * when want_maxima (grid.py:248-277, grid.py:155-162, wcsph.py:239-240,
 * pcisph.py:509-510 where `force` holds f_ext and f_p is added). */
int rts_grid_keys(const RtsParams *p, const RtsBuffers *b, int want_maxima, int add_fp,
                  void *stream);
/* Boundary culling by 1-dilated occupancy, exclusive scan of block counts,
 * stable scatter into (starts, order): fluid ascending then active boundary
 * ascending within each block (grid.py:279-293, _counting_sort grid.py:70-85). */
int rts_grid_sort(const RtsParams *p, const RtsBuffers *b, void *stream);
/* Per-block maxima only (reduce_fluid_max, grid.py:347-351) on current
 * fluid_cells; f_p added to force when add_fp. */
int rts_block_maxima(const RtsParams *p, const RtsBuffers *b, int add_fp, void *stream);

/* ---- region fields (regions.py) -------------------------------------- */
/* assign_regions (regions.py:38-75) then smooth_regions (regions.py:78-91)
 * into block_field; expand_fast_regions (regions.py:94-107) when expand;
 * pin_region override (wcsph.py:258-259, pcisph.py:528-529).  expand=2:
 * assign_regions only (required levels of _mark_timestep_updates). */
int rts_block_levels(const RtsParams *p, const RtsBuffers *b, int expand, void *stream);
/* The public region-field functions on caller-provided fields (regions.py:
 * smooth_regions, expand_fast_regions, derive_observed):
 *   op 0: smooth    block_raw -> block_field
 *   op 1: expand    block_tmp -> block_field over `arg` layers (scratch block_flag, block_raw)
 *   op 2: observed  block_field + error-block mask in block_flag -> block_tmp (0/1)
 *   op 3: neighbour minimum of block_raw, out-of-grid cells = arg -> block_field */
int rts_region_op(const RtsParams *p, const RtsBuffers *b, int op, int arg, void *stream);

/* ---- RTS-PCISPH (pcisph.py) ------------------------------------------- */
/* Wall rows of xs (static positions as fp64, p = -1). */
int rts_pci_walls(const RtsParams *p, const RtsBuffers *b, void *stream);
/* Sorted candidate positions cpos[k] = pos[order[k]] and slot_of, at major
 * start; k_integrate keeps them current so the stale-grid search of later
 * minor steps reads current positions (grid.py:140-143) contiguously. */
int rts_pci_gather(const RtsParams *p, const RtsBuffers *b, void *stream);
/* _assign_major_regions particle tail (pcisph.py:531-534): region, validity
 * = VALIDITY_PERIOD[region], compute = 1, S_e = empty. */
int rts_pci_major_particles(const RtsParams *p, const RtsBuffers *b, void *stream);
/* search_into on the stale major grid for compute/all particles, layers 2
 * for region 1 when two_layer_r1 (grid.py:88-152, pcisph.py:553-557), fused
 * with _ext_forces (pcisph.py:174-199). */
int rts_pci_refresh(const RtsParams *p, const RtsBuffers *b, int all, int two_layer_r1,
                    void *stream);
/* BlockGrid.search_into (grid.py:297-331): rows nbr / cnt for the n particles
 * listed in active, layers[t] block layers for entry t, candidates from cpos
 * (rts_pci_gather of the positions searched). */
int rts_grid_search(const RtsParams *p, const RtsBuffers *b, const int8_t *layers, int n,
                    void *stream);
/* _predict_motion (pcisph.py:202-213): all fluid, or the last force list. */
int rts_pci_motion(const RtsParams *p, const RtsBuffers *b, int all, void *stream);
/* turn | S_e | S_ob membership (pcisph.py:634-643) -> pred list (active),
 * force list (list2); all_pred=1 for the synchronous baselines. */
int rts_pci_sets(const RtsParams *p, const RtsBuffers *b, int row_mask, int all_pred,
                 void *stream);
/* _predict_density + _accumulate_pressure (pcisph.py:216-235, 432-437). */
int rts_pci_density(const RtsParams *p, const RtsBuffers *b, void *stream);
/* S_e = err > eta_max/2 and its blocks (with_se), max err, sum rho*,
 * any(S_e) into the counters (pcisph.py:662, 421-430, 682-683). */
int rts_pci_se_reduce(const RtsParams *p, const RtsBuffers *b, int with_se, void *stream);
/* Static part of derive_observed (regions.py:110-125: occupied and next to
 * a strictly smaller region) into block_tmp; the S_e part (regions.py:123-124)
 * is carried by the generation stamps se_stamp/near_stamp written in
 * rts_pci_se_reduce, and S_ob = static | (near & !S_e) is evaluated per
 * particle (rts_pci_sets, rts_pci_sob, k_integrate).  with_se is ignored. */
int rts_pci_observed(const RtsParams *p, const RtsBuffers *b, int with_se, void *stream);
int rts_pci_sob(const RtsParams *p, const RtsBuffers *b, void *stream);
/* _pressure_forces over the force list (pcisph.py:238-271). */
int rts_pci_pforces(const RtsParams *p, const RtsBuffers *b, void *stream);
/* _integrate (pcisph.py:759-768) + validity countdown (pcisph.py:580-584).
 * countdown bit 0: RTS minor step (countdown, S_ob, candidate copies); bit 1:
 * also the per-block maxima of rts_block_maxima(add_fp = 1) into vmax / fmax,
 * which the caller zeroes first (no ghost rows). */
int rts_pci_integrate(const RtsParams *p, const RtsBuffers *b, int countdown, void *stream);
/* _mark_timestep_updates (pcisph.py:718-755) from the per-block maxima in
 * vmax / fmax: computes the required levels itself (-> block_raw, as
 * rts_block_levels expand = 2 would), then the new field and the particles'
 * regions / validity / compute. */
int rts_pci_mark_updates(const RtsParams *p, const RtsBuffers *b, void *stream);
/* local-phase snapshot (restore=0) / revert (restore=1) of p, f_p (pcisph.py:694-707). */
int rts_pci_snapshot(const RtsParams *p, const RtsBuffers *b, int restore, void *stream);
/* max |v| over fluid into ctr->fmax_bits (_adapt_dt, pcisph.py:470-476). */
int rts_vel_max(const RtsParams *p, const RtsBuffers *b, void *stream);
/* Neighbour audit (count_missing_neighbors, grid.py:165-212, 353-394): `a`
 * describes a grid freshly rebuilt at the current positions (its cpos filled
 * by rts_pci_gather); for every particle of `b`'s refresh list, count the
 * true neighbours (fp64 r^2 < h^2 over one block layer of `a`) absent from
 * its table row; the total goes to b->ctr->missing. */
int rts_pci_audit(const RtsParams *pa, const RtsBuffers *a, const RtsBuffers *b, void *stream);
/* p = f_p = 0 for all fluid (pcisph.py:570-571). */
int rts_pci_zero_pressure(const RtsParams *p, const RtsBuffers *b, void *stream);
/* Device loop control: reset per major; per-minor state reset + first row;
 * per-minor StepStats record into ctl->stats. */
int rts_pci_major_begin(const RtsParams *p, const RtsBuffers *b, void *stream);
int rts_pci_minor_begin(const RtsParams *p, const RtsBuffers *b, int minor, int sync_mode,
                        void *stream);
int rts_pci_minor_end(const RtsParams *p, const RtsBuffers *b, int minor, void *stream);
/* One correction iteration incl. the k_control decision kernel
 * (pcisph.py:633-715; sync_mode: pcisph.py:446-468).  cond_handle: the
 * cudaGraphConditionalHandle of an enclosing while node, or 0. */
int rts_pci_iteration(const RtsParams *p, const RtsBuffers *b, int sync_mode,
                      unsigned long long cond_handle, int local_attempts, int iteration_cap,
                      void *stream);
/* The decision kernel alone (+ snapshot/revert pass in RTS mode). */
int rts_pci_control(const RtsParams *p, const RtsBuffers *b, int sync_mode,
                    unsigned long long cond_handle, int local_attempts, int iteration_cap,
                    void *stream);
/* Minor step before / after the correction loop (pcisph.py:553-587). */
int rts_pci_minor_head(const RtsParams *p, const RtsBuffers *b, int minor, void *stream);
int rts_pci_minor_tail(const RtsParams *p, const RtsBuffers *b, int minor, int last,
                       void *stream);
/* Whole major step (mode 0, n_minor minors) or synchronous step (mode 1) as
 * one CUDA graph with conditional while nodes; NULL + *err on failure. */
void *rts_pci_graph_create(const RtsParams *p, const RtsBuffers *b, int mode, int n_minor,
                           int local_attempts, int iteration_cap, int *err);
int rts_graph_launch(void *graph, void *stream);
void rts_graph_destroy(void *graph);
/* Kernel nodes of a graph: run once per launch / once per correction
 * iteration of each conditional while body (for launch accounting). */
int rts_graph_kernel_counts(void *graph, long long *static_kernels, long long *body_kernels);

/* ---- RTS-WCSPH (wcsph.py) -------------------------------------------- */
/* Validity countdown / pre-emption (wcsph.py:262-266) fused with the sorted
 * candidate gather and the active-list compaction. rts=0: all active. */
int rts_wcsph_propagate(const RtsParams *p, const RtsBuffers *b, void *stream);
/* Density + clamped Tait pressure for active particles (wcsph.py:45-60)
 * over the on-the-fly 3x3x3 block search (grid.py:88-152, layers=1). */
int rts_wcsph_density(const RtsParams *p, const RtsBuffers *b, void *stream);
/* dt_corr/dt_since/acc_prev bookkeeping (wcsph.py:288-290), forces
 * (wcsph.py:63-105) and acc = F/m (wcsph.py:296). */
int rts_wcsph_forces(const RtsParams *p, const RtsBuffers *b, void *stream);
/* Predictor for all, corrector for active, clamp (wcsph.py:299-319). */
/* np.var(rho) over the fluid (wcsph.py:231-232, track_rho_variance): two
 * fixed-order fp64 passes over b->rho using b->partial (>= 513 doubles);
 * *out (device) = the population variance.  Deterministic. */
int rts_rho_variance(const RtsParams *p, const RtsBuffers *b, double *out, void *stream);
int rts_wcsph_integrate(const RtsParams *p, const RtsBuffers *b, void *stream);
/* One whole RTS-WCSPH step as a CUDA graph (launch with rts_graph_launch,
 * destroy with rts_graph_destroy); NULL + *err on failure. */
void *rts_wcsph_graph_create(const RtsParams *p, const RtsBuffers *b, int *err);
/* max |F| over fluid into ctr->fmax_bits (cfl_bound, wcsph.py:182-189). */
int rts_force_max(const RtsParams *p, const RtsBuffers *b, void *stream);

/* ---- x-slab ranks (no reference counterpart: the
 * reference correction loop pcisph.py:612-716 runs in one process) ------- */
#define RTS_HALO_MAX_FIELDS 16
typedef struct {
    void *ptr;              /* storage row 0 of the field */
    const int32_t *remap;   /* row -> storage row (e.g. slot_of), or NULL */
    int32_t words;          /* elements exchanged per row, one message word each
                             * (4-byte elements; fp64 = 2) */
    int32_t stride;         /* elements between consecutive storage rows */
    int32_t msg_off;        /* first word of the field inside a message row */
    int32_t esize;          /* element bytes: 4 (or 0), or 1 for int8 / bool fields
                             * (zero-extended into their message word) */
} RtsHaloField;
typedef struct {
    int32_t n_fields;       /* 1 .. RTS_HALO_MAX_FIELDS */
    int32_t row_words;      /* sum of f[].words (words moved per row) */
    int32_t msg_words;      /* message row width; fields may share words on unpack
                             * (one received word stored in two places) */
    int32_t pad;
    RtsHaloField f[RTS_HALO_MAX_FIELDS];
} RtsHaloSpec;
/* out[r * msg_words + f.msg_off + w] = word w of field f of row rows[r]
 * (r < n), bit copies (fp64 fields travel as two words); rows[r] < 0 is a
 * padding entry (skipped, here and in rts_halo_unpack). */
int rts_halo_pack(const RtsHaloSpec *s, const int32_t *rows, int64_t n, uint32_t *out,
                  void *stream);
/* Inverse of rts_halo_pack: word w of field f of row rows[r] =
 * in[r * msg_words + f.msg_off + w]. */
int rts_halo_unpack(const RtsHaloSpec *s, const int32_t *rows, int64_t n, const uint32_t *in,
                    void *stream);
/* Slab geometry of one rank (block columns along x of the padded grid). */
typedef struct {
    double origin_x, inv_block;   /* grid.py:225-229 */
    int32_t nx;                   /* block columns of the whole grid */
    int32_t lo, hi;               /* owned columns [lo, hi) */
    int32_t halo;                 /* ghost band width in columns */
    int32_t has_left, has_right;  /* neighbour ranks exist */
    int32_t left_lo, right_hi;    /* owned range of the neighbours: [left_lo, lo), [hi, right_hi) */
} RtsSlabGeom;
/* Rows [0, n) of pos (fp32, stride 3), block column as grid.py:248-250, into
 * six lists (row stride list_stride >= n; order free): 0/1 migrants to the
 * left/right neighbour, 2/3 kept rows in the band next to the left/right
 * neighbour, 4/5 migrants inside that neighbour's band next to this slab;
 * leave[i] = 1 for migrants; counts[0..5] list lengths, counts[6] rows
 * beyond a neighbour's slab (an error for the caller). */
int rts_slab_classify(const RtsSlabGeom *g, const float *pos, int n, int32_t *lists,
                      int64_t list_stride, uint8_t *leave, int32_t *counts, void *stream);
/* Hole-filling plan after migration: holes = rows < n_keep with leave set,
 * fill = rows >= n_keep without (equal counts), both lists -1-padded to
 * n_pad entries (rts_halo_pack / unpack skip rows < 0). */
int rts_slab_holes(const uint8_t *leave, int n, int n_keep, int n_pad, int32_t *holes,
                   int32_t *fill, int32_t *counter, void *stream);
#define RTS_CTL_WORDS 5
/* out[0..4] = (max_err, any_se, sum_rho, n_pred, err_flags) of ctr, as fp64. */
int rts_ctl_publish(const RtsBuffers *b, double *out, void *stream);
/* ctr = fold of the all-gathered (world, RTS_CTL_WORDS) publish rows: MAX of
 * max_err (NaN propagates) / any_se, rank-order SUM of sum_rho / n_pred, OR
 * of err_flags into ctr->err_flags (before rts_pci_control), so every rank
 * takes the same done / failed decision. */
int rts_ctl_fold(const RtsBuffers *b, const double *gathered, int world, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* RTS_SPH_H */
