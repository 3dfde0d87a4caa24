/*
 * b200paint.h -- C-ABI of libb200paint.so, the B200-native (sm_100a) drop-in
 * for the reference's `mg-oras` path: reduced full multigrid with the
 * Robin-optimised restricted-additive-Schwarz (ORAS) block smoother for
 * homogeneous-diffusion inpainting (arXiv 2401.06744).
 *
 * The reference (`diffpaint`, pure Python/NumPy) has no FFI boundary of its
 * own; its boundary is the Python API.  Each entry point below names the
 * reference interface it replaces (paths relative to
 * /root/reference/pkg/src/diffpaint/).  INTEGRATION.md shows the ctypes stub a
 * maintainer of the reference would add.
 *
 * Conventions
 *   - plain pointers and sizes only; no C++/torch types cross this boundary;
 *   - every function returns 0 on success, <0 for an argument/usage error,
 *     >0 for a CUDA runtime error code; b200p_last_error() gives the text;
 *   - "d_" pointers are device pointers owned by the caller, "h_" pointers are
 *     host pointers; fields are row-major fp64 (core.py:14-16), masks are one
 *     byte per pixel (0 / non-zero);
 *   - a plan is not thread-safe; different plans may be used concurrently;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *   - there is NO CPU fallback: without a CUDA device every compute entry
 *     point fails with a CUDA error.
 */
#ifndef B200PAINT_H
#define B200PAINT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B200P_MAX_LEVELS 32
#define B200P_ABI_VERSION 2    /* 2: b200p_config lost `spec_cycles`; history_len counts past the cap; image entry points */
#define B200P_MAX_HISTORY 128  /* history entries STORED per report; history_len may be larger (b200p_plan_history has all) */
#define B200P_MAX_BLOCK 64     /* largest supported block edge */

enum {
    B200P_OK = 0,
    B200P_ERR_ARG = -1,         /* ValueError in the reference */
    B200P_ERR_EMPTY_MASK = -2,  /* EmptyMaskError (core.py:28-33, multigrid.py:442-443) */
    B200P_ERR_UNSUPPORTED = -3,
    B200P_ERR_STATE = -4
};

/* MultigridConfig (multigrid.py:50-82) + SolverConfig (solvers.py:43-69) +
 * the problem geometry (InpaintingProblem, core.py:118-166). */
typedef struct b200p_config {
    int width, height, channels;  /* W, H, C of one frame */
    int frames;                   /* frames batched in one plan (independent problems) */
    double spacing;               /* InpaintingProblem.spacing, > 0 */
    int block_size, overlap;      /* MultigridConfig.block_size / overlap */
    int nu_pre, nu_post;          /* smoothing sweeps around the coarse correction */
    int v_cycles_max;             /* MultigridConfig.v_cycles_max */
    int value_downsampling;       /* 1 = "modified", 0 = "naive" */
    double coarse_tol;            /* MultigridConfig.coarse_tol */
    int coarse_max_iters;         /* MultigridConfig.coarse_max_iters */
    double tol_rel;               /* SolverConfig.tol_rel */
    double alpha;                 /* SolverConfig.alpha (Robin weight) */
    double eta;                   /* SolverConfig.local_tol_fraction */
    int local_max_iters;          /* SolverConfig.local_max_iters, 0 = None -> 4*bh*bw */
    int use_graphs;               /* 1: the whole solve is one CUDA graph (WHILE node for the V-cycle loop);
                                     0: eager launches, the host reads the loop condition after every cycle */
    int mode;                     /* MultigridConfig.mode: 0 "full_multigrid" (mg-oras), 1 "multilevel" (ml-oras,
                                     cascade with every level smoothed to tol_rel, multigrid.py:412-418, :449-464),
                                     2 "single": oras_solve on the finest level only (solvers.py:427-485) */
    int max_outer_iters;          /* SolverConfig.max_outer_iters (sweep cap per level in multilevel mode) */
    int smoother;                 /* MultigridConfig.smoother: 0 "oras" (the hot path), 1 "cg" (_cg_run,
                                     solvers.py:97-128: the comparison pipelines cg / ml-cg / mg-cg) */
    int smoother_cg_iters;        /* SolverConfig.smoother_cg_iters: CG steps per smoothing unit */
} b200p_config;

/* SolveReport (solvers.py:72-94), one per (frame, channel). */
typedef struct b200p_report {
    int iterations;               /* V-cycles */
    int converged;
    int fine_smoother_iterations;
    int history_len;              /* values recorded (iterations + 1 for mg-*, one per sweep / step for the
                                     comparison pipelines); only the first B200P_MAX_HISTORY are stored below */
    double final_rel_residual;
    double baseline_residual;
    double init_residual;
    double history[B200P_MAX_HISTORY];
} b200p_report;

typedef struct b200p_level_info {
    int height, width;
    int nx, ny, block_w, block_h;
    double spacing;
} b200p_level_info;

typedef struct b200p_plan b200p_plan;

/* ---- strip mode (single frame over several GPUs; BASELINE config 4b) ----
 * The finest `levels` levels are cut into horizontal strips, one per rank; the coarser levels are
 * replicated.  On a striped level a rank owns the pixel rows [own_lo, own_hi), solves the block
 * rows that cover them (boundary block rows redundantly on both sides), and keeps the halo
 * [ext_lo, ext_hi) of the level's iterate valid.  The library calls `exchange` where data has to
 * move between ranks; kind = base + 16 * (level of the field).  The callback works on `stream`
 * (asynchronously or not) and returns 0 on success:
 *   B200P_XCHG_SUM_RS     d_ptr = (P) doubles: sum over ranks (partial ||r||^2 of the strips)
 *   B200P_XCHG_MAX_FLAGS  d_ptr = (P) ints:    max over ranks
 *   B200P_XCHG_HALO_U     d_ptr = iterate of the level (P,h,w): rows [own_lo, own_hi) are new on
 *                         every rank; fill [ext_lo, own_lo) and [own_hi, ext_hi) from their owners
 *   B200P_XCHG_HALO_RC    the same for the restricted residual of a striped level >= 1
 *   B200P_XCHG_GATHER_RC  d_ptr = restricted residual of the first REPLICATED level (P,h,w): every
 *                         rank wrote the rows [own_lo/2, own_hi/2) of the level above; make the
 *                         whole field identical everywhere (all-gather)
 * Inputs (mask, known) are given in full on every rank; the output holds the rank's rows (plus halo).
 * Strip plans run eagerly (use_graphs = 0).  Needs 32x32 blocks, width % 4 == 0, even block stride. */
enum { B200P_XCHG_SUM_RS = 1, B200P_XCHG_MAX_FLAGS = 2, B200P_XCHG_HALO_U = 3, B200P_XCHG_GATHER_RC = 4,
       B200P_XCHG_HALO_RC = 5 };
typedef int (*b200p_exchange_fn)(void *user, int kind, void *d_ptr, void *stream);
/* Per-step hook of the CG solvers (the `callback` of cg_solve, solvers.py:171-174, and of the "multilevel"
 * mode with the CG smoother, multigrid.py:449-464 / 316-321): called on the calling thread after every CG step
 * of the finest level with the iterate d_u ((frames*C, h, w) fp64 on the device, complete: the solve's stream
 * has been synchronised); a non-zero return aborts the solve. */
typedef int (*b200p_step_fn)(void *user, const double *d_u, int height, int width);

const char *b200p_last_error(void);
/* 1 when the library was built with -DB200P_EXPERIMENTS (block-solve variants that lost their A/B,
 * selected by B200P_TILE32 / B200P_FUSED / B200P_ARRIVAL); the default build does not contain them. */
int b200p_has_experiments(void);
/* B200P_ABI_VERSION of the built library (bindings compare it with the header they were written for). */
int b200p_abi_version(void);
int b200p_device_count(void);
/* CUDA's current device is per host thread: worker threads that drive their own plan
 * (pipeline lanes) select the device of their process first. */
int b200p_set_device(int device);
int b200p_get_device(int *device);

/* Defaults of MultigridConfig()/SolverConfig() for a W x H x C problem. */
void b200p_config_default(b200p_config *cfg, int width, int height, int channels);

/* ---- host-side geometry (no GPU needed) -------------------------------- */

/* partition._axis_starts (partition.py:84-90).  Returns the block count and
 * writes min(count, cap) starts. */
int b200p_axis_starts(int dim, int block, int overlap, int64_t *out, int cap);
/* partition._axis_weights (partition.py:137-154).  w is (n, block_dim) with
 * block_dim = min(block, dim). */
int b200p_axis_weights(int dim, int block, int overlap, double *w, int cap);
/* Level shapes of build_hierarchy (multigrid.py:236-261).  Returns the level
 * count; fills min(count, cap) entries. */
int b200p_level_shapes(int width, int height, double spacing, int block, int overlap,
                       b200p_level_info *out, int cap);

/* ---- plan -------------------------------------------------------------- */

/* Validates the configuration (same ValueError conditions as
 * MultigridConfig.__post_init__, SolverConfig.__post_init__,
 * build_partition), builds level geometry, partition-of-unity tables and all
 * device scratch.  Replaces build_hierarchy's geometry half + Level.__init__
 * (multigrid.py:189-207) + BlockSolver.__init__ (solvers.py:266-301). */
int b200p_plan_create(const b200p_config *cfg, b200p_plan **out);
void b200p_plan_destroy(b200p_plan *plan);
int b200p_plan_num_levels(const b200p_plan *plan);
int b200p_plan_level_info(const b200p_plan *plan, int level, b200p_level_info *out);
/* Strip geometry of rank `rank` of `nranks` on the `levels` finest levels of this plan: the rows are
 * dealt out evenly (cuts at multiples of 2^levels); out[6 * l + ...] = {own_lo, own_hi, ext_lo, ext_hi,
 * iy_lo, iy_hi} of level l.  Host-only. */
int b200p_plan_strip_ranges(const b200p_plan *plan, int levels, int rank, int nranks, int *out);
/* The same from the geometry alone (image height, block_size, overlap). */
int b200p_strip_ranges(int height, int block, int overlap, int levels, int rank, int nranks, int *out);
/* Puts the plan into strip mode on its `levels` finest levels with the given ranges (from
 * b200p_plan_strip_ranges) and callback; rank / nranks themselves are the callback's business.
 * levels = 0 (and a NULL callback) leaves strip mode. */
int b200p_plan_set_strip(b200p_plan *plan, int levels, const int *ranges, b200p_exchange_fn exchange, void *user);
/* Strip mode with the LIBRARY doing the exchanges: `nccl_comm` is an ncclComm_t of `nranks`
 * ranks (this process = `rank`), `ranges_all` the 6 * levels ints of EVERY rank, rank-major, as
 * b200p_strip_ranges writes them.  Per sweep of a striped level the library issues, on the solve's stream,
 *   ncclAllReduce(sum, P doubles) + ncclAllReduce(max, P ints)   after every K1   (global ||r||^2, flags)
 *   ncclGroupStart; ncclSend / ncclRecv of the halo rows; ncclGroupEnd   after every combine
 * and per V-cycle the halo / all-gather of the restricted residual: no host code between the kernels.  With
 * use_graphs = 1 the front part and one V-cycle are captured as two CUDA graphs (collectives included) after
 * one eager warm-up solve; the host reads the loop condition between replays.  libnccl.so.2 is loaded with
 * dlopen on first use (the copy already in the process wins).  levels = 0 leaves strip mode. */
int b200p_plan_set_strip_nccl(b200p_plan *plan, int levels, const int *ranges_all, int rank, int nranks,
                              void *nccl_comm);
/* For hosts without NCCL bindings: ncclGetUniqueId (128 bytes, to be broadcast by the caller),
 * ncclCommInitRank on the current device, ncclCommDestroy. */
int b200p_nccl_unique_id(void *id128);
int b200p_nccl_comm_create(const void *id128, int rank, int nranks, void **nccl_comm);
int b200p_nccl_comm_destroy(void *nccl_comm);
/* The row intervals rank `rank` receives into / sends out of striped level `level` in one halo exchange,
 * as (peer, y0, y1) triples (peer -1 pads the shorter list); returns max(#recv, #send).  Host-only. */
int b200p_strip_halo_plan(const int *ranges_all, int levels, int level, int rank, int nranks, int *recv, int *send,
                          int cap);
/* Device pointer of the level's restricted-residual field (P,h,w) (level >= 1), for the callback. */
int b200p_plan_level_rc(const b200p_plan *plan, int level, double **d_rc);
/* Bytes of device memory the plan holds. */
int64_t b200p_plan_device_bytes(const b200p_plan *plan);
/* Kernel launches issued by the plan since creation (graph replays count the
 * kernel nodes they contain). */
int64_t b200p_plan_launch_count(const b200p_plan *plan);

/* Per-kernel timing for the roofline report.  While enabled, solves run eagerly
 * (no graph replay) with a CUDA event pair around every kernel launch on the
 * launching stream.  `kind` indexes the kernel classes 0..profile_kinds()-1
 * (names from b200p_plan_profile_name); _get returns the accumulated device
 * milliseconds, launch count and algorithmic bytes since enable. */
int b200p_plan_profile(b200p_plan *plan, int enable);
int b200p_plan_profile_kinds(void);
const char *b200p_plan_profile_name(int kind);
int b200p_plan_profile_get(b200p_plan *plan, int kind, double *ms, int64_t *launches, double *bytes);

/* solve_image(problem, "mg-oras", cfg) (pipelines.py:96-114) for `frames`
 * frames at once: d_mask (frames,H,W) bytes, d_known (frames,C,H,W) fp64,
 * d_out (frames,C,H,W) fp64, h_reports frames*C entries (host).  Enqueues on
 * `stream` and synchronises it before returning.  cfg.mode / cfg.smoother select
 * the pipeline: mg-oras (default, the tuned hot path), ml-oras, oras, mg-cg,
 * ml-cg, cg.  The caller must have checked the masks are not empty
 * (b200p_solve_host does). */
int b200p_solve(b200p_plan *plan, const uint8_t *d_mask, const double *d_known, double *d_out,
                b200p_report *h_reports, void *stream);

/* The same solve without the host in the loop: the whole of fmg_solve is ONE CUDA graph
 * (front half -> WHILE node whose body is a V-cycle + convergence check,
 * multigrid.py:474-479, the loop condition is set on the device -> report gather into a
 * pinned host record).  b200p_solve_async only enqueues on `stream`; b200p_solve_wait
 * synchronises that stream and fills h_reports (may be NULL).  One solve may be pending
 * per plan.  b200p_solve == b200p_solve_async + b200p_solve_wait. */
int b200p_solve_async(b200p_plan *plan, const uint8_t *d_mask, const double *d_known, double *d_out,
                      void *stream);
int b200p_solve_wait(b200p_plan *plan, b200p_report *h_reports);

/* Same through HOST buffers: H2D of mask+known, solve, D2H of the result.
 * Returns B200P_ERR_EMPTY_MASK if any frame's mask is all zero. */
int b200p_solve_host(b200p_plan *plan, const uint8_t *h_mask, const double *h_known, double *h_out,
                     b200p_report *h_reports);

/* H2D of the host f64 entry points is SPARSE when the mask is: the path reads `known` only at
 * mask pixels (rhs = where(mask, known, 0), core.py:147-151), so only the mask plane and those values
 * cross PCIe: from a pinned h_known a kernel fetches them in place (zero copy); from a pageable one
 * the call gathers a (pixel index, C values) list into pinned staging and a scatter kernel rebuilds
 * the zero-filled known plane on the device.  Lists larger than half the dense planes,
 * or B200P_DENSE_INGEST=1 in the environment, copy the planes unchanged.  Results are identical.
 * b200p_plan_last_transfer_bytes reports what the last host entry point copied each way. */
int b200p_plan_last_transfer_bytes(const b200p_plan *plan, int64_t *h2d_bytes, int64_t *d2h_bytes);
/* fp64 ingest of the host entry points (results are identical in every mode):
 * mode 0 (default): sparse when the mask is sparse -- from a pinned source the device fetches the values at
 *   mask pixels itself (zero copy; lowest latency of a single solve: 4K RGB 2 %, 9.6 ms vs 12.4 ms host to
 *   host), from a pageable source the library's host threads compact them (mode 2);
 * mode 1: always copy the planes with the copy engine (costs no SM time, overlaps the other lanes' kernels);
 * mode 2: the library's host threads (B200P_HOST_THREADS, default min(8, cores)) compact a (pixel index,
 *   C values) list into pinned staging whatever the source, and a scatter kernel rebuilds the plane: 12 MB
 *   instead of 207 MB per 4K RGB frame on the link and no device reads of host memory -- what a multi-lane
 *   pipeline wants (measured on 5 lanes: 257 frames/s against 230 for mode 1 and 192 for the zero copy of
 *   mode 0, whose reads queue behind the lanes' D2H traffic). */
int b200p_plan_set_ingest(b200p_plan *plan, int mode);

/* 8-bit ingest/egress variant (fileio.image_from_fields, fileio.py:58-65):
 * h_known_u8 (frames,C,H,W) uint8, result rounded half-to-even and clipped to
 * [0,255] on the device.  h_out_u8 (frames,C,H,W). */
int b200p_solve_host_u8(b200p_plan *plan, const uint8_t *h_mask, const uint8_t *h_known_u8,
                        uint8_t *h_out_u8, b200p_report *h_reports);

/* Asynchronous forms of the two host entry points: copies and solve are enqueued on the
 * plan's own stream and the call returns; b200p_solve_wait completes them.  The host buffers
 * must stay valid (and should be pinned for the copies to overlap other plans' kernels)
 * until the wait returns.  This is what the frame pipeline drives, one plan per lane. */
int b200p_solve_host_async(b200p_plan *plan, const uint8_t *h_mask, const double *h_known, double *h_out);
int b200p_solve_host_u8_async(b200p_plan *plan, const uint8_t *h_mask, const uint8_t *h_known_u8,
                              uint8_t *h_out_u8);

/* 8-bit image files as they are on disk, replacing the host-side conversions around
 * solve_image in cli._cmd_inpaint (cli.py:80-95):
 *   h_pixels     (frames,H,W,C) uint8, interleaved as ImageFile.pixels holds them (fileio.py:27-37;
 *                C = 1: (frames,H,W)) -- ImageFile.channel_fields (fileio.py:51-55) runs on the device;
 *   h_mask_bits  (frames,H,ceil(W/8)) the P4 raster of read_mask / write_mask (fileio.py:181-230): rows
 *                padded to whole bytes, most significant bit first, 1 = known pixel; padding bits ignored;
 *   h_out        (frames,H,W,C) uint8 = image_from_fields(solve_image(...).fields).pixels
 *                (fileio.py:58-65: round half to even, clip to [0,255], channels last).
 * The rounding rides on the last post-smoothing combine pass of the finest level (no pass over the fp64
 * result); problems that converge without a V-cycle, and the comparison pipelines, take a tail pass.
 * Errors as b200p_solve_host; an all-zero raster is B200P_ERR_EMPTY_MASK. */
int b200p_solve_host_image_u8(b200p_plan *plan, const uint8_t *h_mask_bits, const uint8_t *h_pixels,
                              uint8_t *h_out, b200p_report *h_reports);
int b200p_solve_host_image_u8_async(b200p_plan *plan, const uint8_t *h_mask_bits, const uint8_t *h_pixels,
                                    uint8_t *h_out);

/* ---- stage entry points (A/B tests against the reference functions) ---- */

/* build_hierarchy's data half (multigrid.py:249-260): coarsen mask and known
 * values down all levels of the plan. */
int b200p_plan_build_hierarchy(b200p_plan *plan, const uint8_t *d_mask, const double *d_known,
                               void *stream);
/* Device pointers of level data after build_hierarchy: mask (frames,h,w)
 * bytes; rhs (frames*C,h,w) fp64 (level 0: NULL, rhs is where(mask,known,0)). */
int b200p_plan_level_ptrs(const b200p_plan *plan, int level, const uint8_t **d_mask,
                          const double **d_rhs);
/* SolveReport.history of problem `problem` (frame * C + channel) of the plan's last completed solve, whole:
 * the reference never truncates it (solvers.py:60-75), the b200p_report record keeps only its first
 * B200P_MAX_HISTORY values.  The plan's device buffer is sized from the config's iteration caps
 * (v_cycles_max + 2; max(max_outer_iters, coarse_max_iters) + 2 for the ml- and single-level pipelines).
 * Copies min(cap, stored capacity) doubles to h_out and returns that count (< 0: error); the valid prefix
 * is report.history_len long. */
int b200p_plan_history(b200p_plan *plan, int problem, double *h_out, int cap);
/* Installs (fn != NULL) or removes the per-step hook; it applies to the solves of `cg` and `ml-cg` plans
 * (config.smoother 1, mode 2 / 1), which then check their stop test on the host after every step. */
int b200p_plan_set_step_callback(b200p_plan *plan, b200p_step_fn fn, void *user);
/* cascadic_init (multigrid.py:374-386) after build_hierarchy; d_u (frames*C,H,W).
 * Both stage calls below smooth with config.smoother (ORAS sweeps or CG steps,
 * multigrid.py:264-279). */
int b200p_plan_cascade(b200p_plan *plan, double *d_u, void *stream);
/* v_cycle(hier, level, u, rhs, cfg, counters) (multigrid.py:335-371): one
 * V-cycle at `level` on d_u/d_rhs (frames*C planes of that level's shape),
 * after build_hierarchy.  fine_units (host, frames*C, may be NULL) receives
 * the finest-level smoothing units when level == 0. */
int b200p_plan_vcycle(b200p_plan *plan, int level, double *d_u, const double *d_rhs,
                      int *h_fine_units, void *stream);
/* fmg_solve's second half after cascade: not exposed separately; use b200p_solve. */

/* oras_sweeps(op, blocks, b, u, max_sweeps=, stop_norm=, eta=, local_max_iters=)
 * (solvers.py:393-424) on level `level` of the plan (after build_hierarchy for
 * the masks), d_u/d_b (frames*C planes).  Per problem: sweeps done and final
 * residual norm (host arrays, frames*C).  path: 0 plan default (lean 32x32
 * kernel + combine where the level is eligible), 1 generic shared-memory
 * kernel + combine, 2 register-tile kernel + combine, 3 fused persistent sweep
 * (plans created with B200P_FUSED=1), 10+t tile variant t (DESIGN.md lists
 * them); an ineligible level gives B200P_ERR_UNSUPPORTED. */
int b200p_plan_oras_sweeps(b200p_plan *plan, int level, const double *d_b, double *d_u,
                           int max_sweeps, double stop_norm, int path, int *h_sweeps,
                           double *h_rn, void *stream);
/* BlockSolver.gather + solve_blocks (solvers.py:303-305, :372-390) on a given
 * residual field d_r, target_sq as in the reference; d_v (frames*C, nblocks,
 * bh, bw) receives the UNWEIGHTED local corrections.  Generic kernel only. */
int b200p_plan_solve_blocks(b200p_plan *plan, int level, const double *d_r, double target_sq,
                            double *d_v, void *stream);

/* BlockSolver.scatter_weighted (solvers.py:307-314): d_v (frames*C, nblocks, bh, bw) UNWEIGHTED local
 * corrections -> d_field (frames*C, h, w) = sum_i R_i^T ((v_i * wy_i) * wx_i), summed per pixel in ascending
 * block order like np.bincount.  Runs the sweeps' own combine kernel (K2b) on a zero field, in isolation. */
int b200p_plan_scatter_weighted(b200p_plan *plan, int level, const double *d_v, double *d_field, void *stream);

/* StencilOperator.apply / residual (core.py:100-110) on one (h,w) field. */
int b200p_apply(const uint8_t *d_mask, int h, int w, double spacing, const double *d_u,
                double *d_out, void *stream);
int b200p_residual(const uint8_t *d_mask, int h, int w, double spacing, const double *d_b,
                   const double *d_u, double *d_r, void *stream);
/* ||b - A u||^2 per plane (planes fields sharing one mask). */
int b200p_residual_sqnorm(const uint8_t *d_mask, int h, int w, double spacing, const double *d_b,
                          const double *d_u, int planes, double *h_out, void *stream);

/* Transfers (multigrid.py:98-186); coarse shapes are ceil(h/2) x ceil(w/2). */
int b200p_downsample_mask(const uint8_t *d_fine, int h, int w, uint8_t *d_coarse, void *stream);
/* image_from_fields (fileio.py:58-65): (frames,C,h,w) fp64 -> (frames,h,w,C) uint8, np.round (half to
 * even) then clip to [0,255]; the quantiser the solve's 8-bit egress uses. */
int b200p_image_from_fields(const double *d_fields, int frames, int channels, int h, int w, uint8_t *d_pixels,
                            void *stream);
/* read_mask's P4 branch (fileio.py:206-216): raster rows of ceil(w/8) bytes, MSB first -> (frames,h,w) bytes. */
int b200p_unpack_mask_bits(const uint8_t *d_bits, int frames, int h, int w, uint8_t *d_mask, void *stream);
int b200p_downsample_values(const uint8_t *d_fine_mask, const uint8_t *d_coarse_mask,
                            const double *d_fine_rhs, int h, int w, int modified,
                            double *d_coarse_rhs, void *stream);
/* residual + restrict_residual fused (multigrid.py:358-360). */
int b200p_residual_restrict(const uint8_t *d_fine_mask, const uint8_t *d_coarse_mask, int h, int w,
                            double spacing, const double *d_b, const double *d_u,
                            double *d_coarse_r, void *stream);
/* restrict_residual alone on a given fine residual field (multigrid.py:149-154). */
int b200p_restrict_residual(const double *d_fine_r, const uint8_t *d_coarse_mask, int h, int w,
                            double *d_coarse_r, void *stream);
/* u += prolongate_correction(e, mask) (multigrid.py:367, :175-177). */
int b200p_prolongate_correct(const double *d_coarse_e, const uint8_t *d_fine_mask, int h, int w,
                             double *d_u, void *stream);
/* u = prolongate_solution(coarse_u, mask, rhs) (multigrid.py:180-186). */
int b200p_prolongate_solution(const double *d_coarse_u, const uint8_t *d_fine_mask,
                              const double *d_fine_rhs, int h, int w, double *d_u, void *stream);

/* ---- small device-memory helpers for host languages without a CUDA binding */
int b200p_malloc(void **d_ptr, int64_t bytes);
int b200p_free(void *d_ptr);
/* CUDA IPC for the strip mode's peer-memory transport: export a cudaMalloc'ed buffer (its BASE pointer),
 * map a peer's buffer into this process (reads and writes then go over NVLink / peer memory), unmap it. */
int b200p_ipc_export(const void *d_ptr, unsigned char handle[64]);
int b200p_ipc_open(const unsigned char handle[64], void **d_ptr);
int b200p_ipc_close(void *d_ptr);
int b200p_memcpy_d2d_async(void *d_dst, const void *d_src, int64_t bytes, void *stream);
int b200p_memcpy_h2d(void *d_dst, const void *h_src, int64_t bytes);
int b200p_memcpy_d2h(void *h_dst, const void *d_src, int64_t bytes);
int b200p_memset(void *d_ptr, int value, int64_t bytes);
int b200p_device_synchronize(void);

#ifdef __cplusplus
}
#endif
#endif /* B200PAINT_H */
