// b200paint.cu -- host driver + C-ABI of libb200paint.so (sm_100a only).
//
// Implements include/b200paint.h: plan construction (level geometry, partition
// of unity tables, device scratch), the FMG / V-cycle driver of the reference's
// mg-oras path (multigrid.py:335-487, pipelines.py:96-114) as CUDA-graph
// replays, and stage-level entry points for A/B tests against the reference
// functions.  Frames x channels are batched as independent "problems" p.
//
// There is no CPU fallback anywhere in this file: every compute entry point
// launches CUDA kernels and returns the CUDA error if no device is present.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <dlfcn.h>
#include <nccl.h>   // types only: the library is loaded with dlopen when a strip plan asks for it

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/b200paint.h"
#include "kernels_stencil.cuh"
#include "kernels_rows.cuh"
#include "kernels_rows_tma.cuh"
#include "kernels_oras.cuh"
#include "kernels_oras_warp.cuh"
// Block-solve variants that lost their A/B are compiled only on request:
//   make EXTRA=-DB200P_EXPERIMENTS
#ifdef B200P_EXPERIMENTS
#include "kernels_oras_lab.cuh"
#include "kernels_oras_tma.cuh"
#define B200P_LAB 1
#else
#define B200P_LAB 0
#endif
#include "kernels_cg.cuh"

using namespace b200p;

// ------------------------------------------------------------- errors ------
static thread_local std::string g_err;

static int fail_arg(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

static int fail_cuda(cudaError_t e, const char *what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return (int)e > 0 ? (int)e : 999;
}

#define CU(x)                                            \
    do {                                                 \
        cudaError_t e__ = (x);                           \
        if (e__ != cudaSuccess) return fail_cuda(e__, #x); \
    } while (0)

// ------------------------------------------------------------ geometry -----
// partition._axis_starts (partition.py:84-90)
static std::vector<int> axis_starts(int dim, int block, int stride) {
    std::vector<int> s;
    if (dim <= block) {
        s.push_back(0);
        return s;
    }
    const int count = (dim - block + stride - 1) / stride + 1;
    for (int i = 0; i < count; ++i) s.push_back(stride * i);
    s[count - 1] = dim - block;
    return s;
}

// partition._axis_weights (partition.py:137-154); block = min(block_size, dim).
static std::vector<double> axis_weights(const std::vector<int> &starts, int block, int dim,
                                        int overlap) {
    const int n = (int)starts.size();
    std::vector<double> w((size_t)n * block, 1.0);
    if (overlap > 0) {
        // np.linspace(0, 1, overlap): k * step, endpoint forced to 1; [0.0] for overlap == 1
        std::vector<double> ramp(overlap);
        if (overlap == 1) {
            ramp[0] = 0.0;
        } else {
            const double step = 1.0 / (double)(overlap - 1);
            for (int k = 0; k < overlap; ++k) ramp[k] = (double)k * step;
            ramp[overlap - 1] = 1.0;
        }
        for (int i = 0; i < n; ++i) {
            if (starts[i] > 0)
                for (int k = 0; k < overlap && k < block; ++k) w[(size_t)i * block + k] *= ramp[k];
            if (starts[i] + block < dim)
                for (int k = 0; k < overlap && k < block; ++k)
                    w[(size_t)i * block + block - overlap + k] *= ramp[overlap - 1 - k];
        }
    }
    std::vector<double> total(dim, 0.0);
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < block; ++k) total[starts[i] + k] += w[(size_t)i * block + k];
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < block; ++k) w[(size_t)i * block + k] /= total[starts[i] + k];
    return w;
}

// first covering block and number of covering blocks of every pixel on an axis
static void axis_cover(const std::vector<int> &starts, int block, int dim, std::vector<int> &first,
                       std::vector<int> &count) {
    first.assign(dim, 0);
    count.assign(dim, 0);
    for (int i = (int)starts.size() - 1; i >= 0; --i)
        for (int k = 0; k < block; ++k) {
            first[starts[i] + k] = i;
            count[starts[i] + k] += 1;
        }
}

static int level_shapes(int width, int height, double spacing, int block, int overlap,
                        std::vector<b200p_level_info> &out) {
    int h = height, w = width;
    const int stride = block - overlap;
    for (;;) {
        b200p_level_info L;
        L.height = h;
        L.width = w;
        L.block_w = std::min(block, w);
        L.block_h = std::min(block, h);
        L.nx = (int)axis_starts(w, block, stride).size();
        L.ny = (int)axis_starts(h, block, stride).size();
        L.spacing = spacing;
        out.push_back(L);
        if (std::max(h, w) <= block || (int)out.size() >= B200P_MAX_LEVELS) break;
        h = (h + 1) / 2;
        w = (w + 1) / 2;
        spacing *= 2.0;
    }
    return (int)out.size();
}

// --------------------------------------------------------------- plan ------
enum KernelKind {
    KK_NORM = 0,      // K1
    KK_SWEEP,         // K2F fused sweep
    KK_SWEEP_SPLIT,   // K2 / K2g (split path)
    KK_COMBINE,       // K2b
    KK_RESTRICT,      // K3
    KK_PROLONG_CORR,  // K4
    KK_PROLONG_SOL,   // K5
    KK_DOWN_MASK,     // K6a
    KK_DOWN_VALUES,   // K6b
    KK_COARSE,        // K7
    KK_CONTROL,       // per-problem bookkeeping
    KK_CONVERT,       // u8 ingest / egress
    KK_CG,            // global CG field kernels (comparison pipelines)
    KK_COUNT
};

static const char *const kKindNames[KK_COUNT] = {
    "residual_sqnorm", "oras_sweep", "oras_sweep_split", "oras_combine", "residual_restrict", "prolongate_correct",
    "prolongate_solution", "downsample_mask", "downsample_values", "coarse_solve", "control",
    "convert_u8", "global_cg"};

struct LevelHost {
    b200p_level_info info;
    int nblocks = 0;
    LevelDev dev;
    uint8_t *d_mask = nullptr;  // (F,h,w); level 0: caller's pointer
    double *d_rhs = nullptr;    // (P,h,w) hierarchy values; level 0: caller's `known`
    double *d_u = nullptr;      // (P,h,w) cascade iterate / V-cycle correction (levels >= 1)
    double *d_rc = nullptr;     // (P,h,w) restricted residual (levels >= 1)
    int tile = 0;               // K2 variant: 0 generic, else see launch_sweep
    unsigned *d_mtab = nullptr; // K2T: packed block-local masks (F, nblocks, 64); null = level not eligible
    unsigned *d_mtabw = nullptr; // K2W: the same for the warp-per-block layout (F, nblocks, 32)
    unsigned *d_claim = nullptr; // K2W: {next unclaimed item, finished CTAs}, zero between launches
    // band combine (K2W DIRECT + oras_combine_band_kernel): per-axis writer tables, row / column lists
    bool band = false;
    const uint8_t *d_xflag = nullptr, *d_yflag = nullptr;
    const int *d_nzxf = nullptr, *d_nzxn = nullptr, *d_nzyf = nullptr, *d_nzyn = nullptr;
    const int *d_band_rows = nullptr, *d_core_rows = nullptr, *d_band_cols = nullptr;
    int n_band_rows = 0, n_core_rows = 0, n_band_cols = 0;
    // combine on arrival (FUSE variant of the lean kernel): cell tables and arrival counters
    const int *d_cell_need = nullptr, *d_lastx = nullptr, *d_lasty = nullptr;
    unsigned *d_cell_cnt = nullptr;
    // strip mode (level 0 only): rows this rank owns / keeps valid, block rows it solves (default: all)
    int own_lo = 0, own_hi = 0, ext_lo = 0, ext_hi = 0, iy_lo = 0, iy_hi = 0;
    bool is_strip = false;
    // fused sweep (K2F): ping-pong partner of the iterate, L2-resident ring, schedule tables
    bool fused = false;
    int fused_tile = 0;
    double *d_u_alt = nullptr;  // (P,h,w)
    double *d_ring = nullptr;   // (R, nx, bh*bw)
    int R = 0, lag = 0, nsx = 0, nc = 0, cw = 0, fused_grid = 0;
    const int *d_band_first_row = nullptr, *d_row_last_band = nullptr;
};

// NVTX range around the launches of one stage of one level ("cascade L3", "vcycle L0 pre", ...): shows up in
// nsys / ncu timelines of eager runs and of graph capture; a no-op without a profiler attached.
struct NvtxScope {
    NvtxScope(const char *what, int level) {
        char buf[48];
        snprintf(buf, sizeof buf, "%s L%d", what, level);
        nvtxRangePushA(buf);
    }
    ~NvtxScope() { nvtxRangePop(); }
};

// current iterate of a level + its ping-pong partner (fused sweeps swap them)
struct UBuf {
    double *cur, *alt;
};

struct ProfEvent {
    int kind;
    double bytes;
    cudaEvent_t a, b;
};

// SolveReport fields of all problems into one (mapped, pinned) host record.
struct ReportPack {
    int *cycles, *units, *histlen;
    double *baseline, *rel, *hist;
};

struct GraphSlot {
    cudaGraphExec_t exec = nullptr;
    const void *k0 = nullptr, *k1 = nullptr, *k2 = nullptr, *k3 = nullptr;  // pointers baked into the graph
    int64_t kernels = 0;
};

struct b200p_plan {
    b200p_config cfg;
    int F = 0, C = 0, P = 0;
    std::vector<LevelHost> lev;
    std::vector<void *> owned;  // device allocations
    int64_t dev_bytes = 0;
    int64_t launches = 0;
    int64_t *launch_sink = nullptr;  // where launches are counted (graph capture: the slot)
    // sweep scratch + norm reduction
    double *d_scratch = nullptr;
    int norm_ctas = 0;
    double *d_partial = nullptr;
    int *d_partial_flag = nullptr;
    unsigned *d_counter = nullptr;
    double *d_rs = nullptr;
    int *d_mflag = nullptr;
    // per-problem FMG control (multigrid.py:466-486)
    int *d_active = nullptr, *d_cycles = nullptr, *d_units = nullptr, *d_histlen = nullptr;
    int *d_any = nullptr;
    double *d_baseline = nullptr, *d_denom = nullptr, *d_rel = nullptr, *d_hist = nullptr;
    unsigned long long *d_stats = nullptr;  // B200P_STATS=1: K2F cycle accounting
    unsigned *d_sched = nullptr;  // K2F counters: [work | row_done P*ny | band_done P*ny]
    size_t sched_words = 0;
    int *d_gate = nullptr, *d_sweeps = nullptr;  // stage API (oras_sweeps with stop_norm)
    double *d_rn = nullptr;
    int *h_any = nullptr;  // pinned
    // single-graph solve: WHILE node handle, pinned report record, pending state
    cudaGraphConditionalHandle cond = 0;
    bool cond_capture = false;   // control kernels drive the WHILE node (set during capture)
    void *h_rep = nullptr;       // mapped pinned host block behind `rep`
    ReportPack rep = {};
    cudaStream_t aux_stream = nullptr;  // captures the WHILE body
    cudaStream_t pending_stream = nullptr;
    bool pending = false;
    bool pending_eager = false;  // the pending solve ran eagerly (launches already counted)
    // strip mode: the finest level is cut into horizontal strips over ranks; `exchange` moves data
    bool strip = false;
    b200p_exchange_fn exchange = nullptr;
    void *exchange_user = nullptr;
    int hist_cap = B200P_MAX_HISTORY;     // values per problem in d_hist (sized from the config's iteration caps)
    b200p_step_fn step_cb = nullptr;      // per-step hook of the recording CG runs (cg / ml-cg callbacks)
    void *step_user = nullptr;
    // native strip exchange: NCCL calls issued by the library on the solve's stream (capturable)
    ncclComm_t nccl_comm = nullptr;
    int nccl_rank = 0, nccl_nranks = 1, strip_levels = 0;
    bool nccl_warm = false;               // one eager solve has run (NCCL connects peers lazily, outside capture)
    std::vector<int> ranges_all;          // [rank][level][6] as b200p_strip_ranges writes them
    // CG-smoothed pipelines (cg, ml-cg, mg-cg): CG vectors sized for level 0 + per-problem state
    double *cg_r = nullptr, *cg_p = nullptr, *cg_q = nullptr;
    CgState cgs = {};
    GraphSlot g_solve;
    int64_t cycle_kernels = 0;   // kernel nodes of one WHILE body pass
    // staging for the host entry points
    uint8_t *d_in_mask = nullptr;
    double *d_in_known = nullptr, *d_out = nullptr;
    uint8_t *d_io_u8 = nullptr;
    uint8_t *d_mask_bits = nullptr;       // P4 raster of the image entry points (F, h, ceil(w / 8))
    // 8-bit egress of the solve being enqueued: target image (F, h, w, C), the sweep that carries it
    bool u_zero_now = false;              // the next sweep's iterate is an implicit zero field (not to be read)
    uint8_t *egress = nullptr, *egress_now = nullptr;
    const double *egress_src = nullptr;   // the fp64 result the tail pass converts
    bool egress_fused = false;            // a combine pass of the cycle body writes the image
    // sparse ingest (host f64 entry point): pixel indices + values at mask pixels, pinned + device
    uint32_t *h_sp_idx = nullptr, *d_sp_idx = nullptr;
    double *h_sp_val = nullptr, *d_sp_val = nullptr;
    size_t sp_cap = 0;
    int64_t last_h2d = 0, last_d2h = 0;  // bytes the last host entry point copied each way
    int ingest_mode = 0;                  // 0 auto (sparse when the mask is), 1 always the dense plane copy, 2 sparse by host gather
    bool last_h2d_counted = false;        // ... H2D side = mask planes + *h_cnt values (counted on the device)
    unsigned long long *h_cnt = nullptr, *d_cnt = nullptr;
    void *h_pin = nullptr;  // pinned bounce buffer
    size_t h_pin_bytes = 0;
    cudaStream_t own_stream = nullptr;
    bool hierarchy_ready = false;
    // graphs
    GraphSlot g_front, g_cycle;
    // profiling
    bool profiling = false;
    std::vector<ProfEvent> prof_events;
    double prof_ms[KK_COUNT] = {0};
    double prof_bytes[KK_COUNT] = {0};
    int64_t prof_launches[KK_COUNT] = {0};
};

template <class T>
static int dev_alloc(b200p_plan *pl, T **out, size_t count) {
    void *p = nullptr;
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    CU(cudaMalloc(&p, bytes));
    pl->owned.push_back(p);
    pl->dev_bytes += (int64_t)bytes;
    *out = reinterpret_cast<T *>(p);
    return 0;
}

template <class T>
static int dev_upload(b200p_plan *pl, const std::vector<T> &v, const T **out) {
    T *d = nullptr;
    int rc = dev_alloc(pl, &d, v.size());
    if (rc) return rc;
    CU(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    *out = d;
    return 0;
}

// Launch bracket: counts the launch, and in profiling mode wraps it in a CUDA
// event pair on the launching stream.
struct LaunchScope {
    b200p_plan *pl;
    cudaStream_t st;
    int idx = -1;
    LaunchScope(b200p_plan *p, cudaStream_t s, int kind, double bytes) : pl(p), st(s) {
        if (pl->launch_sink) *pl->launch_sink += 1; else pl->launches += 1;
        if (pl->profiling) {
            ProfEvent e;
            e.kind = kind;
            e.bytes = bytes;
            cudaEventCreate(&e.a);
            cudaEventCreate(&e.b);
            cudaEventRecord(e.a, st);
            pl->prof_events.push_back(e);
            idx = (int)pl->prof_events.size() - 1;
        }
    }
    ~LaunchScope() {
        if (idx >= 0) cudaEventRecord(pl->prof_events[idx].b, st);
    }
};

static void prof_collect(b200p_plan *pl) {
    for (auto &e : pl->prof_events) {
        float ms = 0.f;
        cudaEventSynchronize(e.b);
        cudaEventElapsedTime(&ms, e.a, e.b);
        pl->prof_ms[e.kind] += ms;
        pl->prof_bytes[e.kind] += e.bytes;
        pl->prof_launches[e.kind] += 1;
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    pl->prof_events.clear();
}

// ------------------------------------------------- control kernels ---------
// fmg_solve bookkeeping (multigrid.py:446, :468-479), one thread per problem.
// stage 0: baseline = sqrt(rs)            (flat-init defect)
// stage 1: first check after the cascade  (denom, rel, history[0], active)
// stage 2: check after a V-cycle          (cycles+1, rel, history, active)
__global__ void fmg_control_kernel(int P, int stage, const double *rs, double tol, int cycles_max,
                                   double *baseline, double *denom, double *rel, double *hist,
                                   int *histlen, int *active, int *cycles, int *units, int *any,
                                   int use_cond, cudaGraphConditionalHandle cond, int hist_cap) {
    // one CTA, problems strided over its threads: the "is any problem still active" verdict is
    // a CTA-wide OR, written to `any` (eager host loop) or to the WHILE node of the solve graph
    int mine = 0;
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
        const double rn = sqrt(rs[p]);
        if (stage == 0) {
            baseline[p] = rn;
            units[p] = 0;
            cycles[p] = 0;
            histlen[p] = 0;
            active[p] = 1;
            continue;
        }
        if (stage == 1) {
            const double base = baseline[p];
            const double d = base > 0.0 ? base : (rn > 0.0 ? rn : 1.0);
            denom[p] = d;
            const double r = rn / d;
            rel[p] = r;
            hist[(size_t)p * hist_cap] = r;
            histlen[p] = 1;
            const int act = (r > tol && 0 < cycles_max) ? 1 : 0;
            active[p] = act;
            mine |= act;
            continue;
        }
        if (!active[p]) continue;
        const int c = cycles[p] + 1;
        cycles[p] = c;
        const double r = rn / denom[p];
        rel[p] = r;
        const int hl = histlen[p];   // counts every recorded value; the plan sizes hist_cap for its config
        if (hl < hist_cap) hist[(size_t)p * hist_cap + hl] = r;
        histlen[p] = hl + 1;
        const int act = (r > tol && c < cycles_max) ? 1 : 0;
        active[p] = act;
        mine |= act;
    }
    if (stage == 0) return;
    const int all = __syncthreads_or(mine);
    if (threadIdx.x == 0) {
        *any = all;
        if (use_cond) cudaGraphSetConditional(cond, all ? 1u : 0u);
    }
}

// SolveReport fields of all problems into one (mapped, pinned) host record.
__global__ void pack_reports_kernel(int P, const int *cycles, const int *units, const int *histlen,
                                    const double *baseline, const double *rel, const double *hist,
                                    int hist_cap, ReportPack out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < P) {
        out.cycles[i] = cycles[i];
        out.units[i] = units[i];
        out.histlen[i] = histlen[i];
        out.baseline[i] = baseline[i];
        out.rel[i] = rel[i];
    }
    // the report record keeps the first B200P_MAX_HISTORY values of each problem (b200p_plan_history: all)
    if (i < P * B200P_MAX_HISTORY)
        out.hist[i] = hist[(size_t)(i / B200P_MAX_HISTORY) * hist_cap + i % B200P_MAX_HISTORY];
}

__global__ void set_int_kernel(int *p, int n, int v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// oras_sweeps exit test (solvers.py:416-421) for the stage API.
__global__ void sweep_gate_kernel(int P, const double *rs, double stop_norm, int max_sweeps,
                                  int *gate, const int *sweeps, double *rn_out, int *any) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P || !gate[p]) return;
    const double r2 = rs[p];
    const double rn = sqrt(r2);
    rn_out[p] = rn;
    if (r2 == 0.0 || rn <= stop_norm || sweeps[p] >= max_sweeps) gate[p] = 0;
    else atomicOr(any, 1);
}

// Multilevel mode (ml-oras): _smooth_to_tol on one level of the cascade (multigrid.py:282-332).
// base: the level's flat-init defect -> denom (0 -> the first residual norm, and 0 again -> done).
__global__ void ml_level_begin_kernel(int P, const double *rs_base, double *denom, int *gate, int *sweeps) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    denom[p] = sqrt(rs_base[p]);
    gate[p] = 1;
    sweeps[p] = 0;
}
// One residual evaluation of oras_sweeps with stop_norm = tol * denom (solvers.py:413-421):
// records the relative norm (history on the finest level), closes the gate on exit.
__global__ void ml_gate_kernel(int P, const double *rs, double tol, int max_units, double *denom, int *gate,
                               const int *sweeps, double *rel, double *hist, int *histlen, int record,
                               int *any, int hist_cap) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P || !gate[p]) return;
    const double r2 = rs[p];
    const double rn = sqrt(r2);
    double d = denom[p];
    if (d == 0.0) {  // multigrid.py:300-303
        d = rn;
        denom[p] = d;
        if (d == 0.0) {
            rel[p] = 0.0;
            gate[p] = 0;
            return;
        }
    }
    const double r = rn / d;
    rel[p] = r;
    if (record) {
        const int hl = histlen[p];   // counts every recorded value; the plan sizes hist_cap for its config
        if (hl < hist_cap) hist[(size_t)p * hist_cap + hl] = r;
        histlen[p] = hl + 1;
    }
    if (r2 == 0.0 || rn <= tol * d || sweeps[p] >= max_units) gate[p] = 0;
    else atomicOr(any, 1);
}
// report fields of multilevel mode: iterations = finest-level smoother units
__global__ void ml_finish_kernel(int P, const int *sweeps, int *cycles, int *units, int *active) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    cycles[p] = sweeps[p];
    units[p] = sweeps[p];
    active[p] = 0;
}

// ------------------------------------------------------ launch helpers -----
static inline dim3 grid2x(int wc, int hc, int z) { return dim3((wc + 63) / 64, (hc + 3) / 4, z); }

// K6a with 8 coarse cells per thread: fine rows are whole 16-byte words, coarse rows whole 8-byte words
static bool words8_ok(int w, const void *fmask, const void *cmask) {
    static const bool want = !(getenv("B200P_K6_WORDS") && atoi(getenv("B200P_K6_WORDS")) == 0);
    return want && w % 16 == 0 && ((uintptr_t)fmask % 16) == 0 && ((uintptr_t)cmask % 8) == 0;
}

static double field_bytes(const b200p_plan *pl, const LevelHost &L, double fields, double masks) {
    const double n = (double)L.info.height * L.info.width;
    return fields * pl->P * 8.0 * n + masks * pl->F * n;
}

static int rows_chunk(int h) { return h >= 1024 ? 32 : (h >= 256 ? 16 : 8); }

// Strip mode: level 0 is cut into horizontal strips over ranks, coarser levels are replicated.
static bool striped(const b200p_plan *pl, const LevelHost &L) { return pl->strip && L.is_strip; }
static int level_of(const b200p_plan *pl, const LevelHost &L) { return (int)(&L - &pl->lev[0]); }

// ---- NCCL, loaded on demand (no link-time dependency: frame sharding never needs it) ----
struct NcclApi {
    void *handle = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int *) = nullptr;
    ncclResult_t (*CommUserRank)(const ncclComm_t, int *) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi *nccl_api() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        // the copy already in the process (torch loads its own) wins, then the system library
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            bool ok = true;
#define NCCL_SYM(field, name) ok = ok && ((*(void **)(&api.field) = dlsym(h, name)) != nullptr)
            NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
            NCCL_SYM(CommInitRank, "ncclCommInitRank");
            NCCL_SYM(CommDestroy, "ncclCommDestroy");
            NCCL_SYM(CommCount, "ncclCommCount");
            NCCL_SYM(CommUserRank, "ncclCommUserRank");
            NCCL_SYM(AllReduce, "ncclAllReduce");
            NCCL_SYM(Send, "ncclSend");
            NCCL_SYM(Recv, "ncclRecv");
            NCCL_SYM(GroupStart, "ncclGroupStart");
            NCCL_SYM(GroupEnd, "ncclGroupEnd");
            NCCL_SYM(GetErrorString, "ncclGetErrorString");
#undef NCCL_SYM
            if (ok) api.handle = h;
        }
    }
    return api.handle ? &api : nullptr;
}

#define NC(x)                                                                                        \
    do {                                                                                             \
        ncclResult_t r__ = (x);                                                                      \
        if (r__ != ncclSuccess) return fail_arg(B200P_ERR_STATE, "%s: %s", #x, N->GetErrorString(r__)); \
    } while (0)

// Row intervals of a halo exchange on one striped level, seen from rank `me`: what it receives into its halo
// [ext_lo, own_lo) + [own_hi, ext_hi) from the owners of those rows, and what it sends out of its own rows into
// the halos of the others.  Both sides enumerate a pair's intervals from the RECEIVER's ranges (halo above,
// then halo below), so sends and receives of a pair match in order.
struct RowMove {
    int peer, y0, y1;
};
static void halo_moves(const int *ranges_all, int levels, int level, int me, int nranks, std::vector<RowMove> &recv,
                       std::vector<RowMove> &send) {
    auto rg = [&](int q) { return ranges_all + ((size_t)q * levels + level) * 6; };
    auto cut = [](const int *to, const int *from, int peer, std::vector<RowMove> &out) {
        // rows of `to`'s halo that `from` owns
        const int parts[2][2] = {{to[2], to[0]}, {to[1], to[3]}};
        for (const auto &pr : parts) {
            const int a = std::max(pr[0], from[0]), b = std::min(pr[1], from[1]);
            if (a < b) out.push_back({peer, a, b});
        }
    };
    recv.clear();
    send.clear();
    for (int q = 0; q < nranks; ++q) {
        if (q == me) continue;
        cut(rg(me), rg(q), q, recv);
        cut(rg(q), rg(me), q, send);
    }
}

// The exchanges of include/b200paint.h (B200P_XCHG_*) as NCCL calls on `st`.
static int strip_exchange_nccl(b200p_plan *pl, int base, int level, void *d_ptr, cudaStream_t st) {
    NcclApi *N = nccl_api();
    if (!N) return fail_arg(B200P_ERR_STATE, "libnccl.so.2 could not be loaded");
    const int P = pl->P, me = pl->nccl_rank, nr = pl->nccl_nranks;
    if (base == B200P_XCHG_SUM_RS) {
        NC(N->AllReduce(d_ptr, d_ptr, (size_t)P, ncclDouble, ncclSum, pl->nccl_comm, st));
        return 0;
    }
    if (base == B200P_XCHG_MAX_FLAGS) {
        NC(N->AllReduce(d_ptr, d_ptr, (size_t)P, ncclInt32, ncclMax, pl->nccl_comm, st));
        return 0;
    }
    if (nr == 1) return 0;
    const LevelHost &L = pl->lev[level];
    const size_t w = (size_t)L.info.width, plane = w * L.info.height;
    double *f = static_cast<double *>(d_ptr);
    if (base == B200P_XCHG_HALO_U || base == B200P_XCHG_HALO_RC) {
        std::vector<RowMove> recv, send;
        halo_moves(pl->ranges_all.data(), pl->strip_levels, level, me, nr, recv, send);
        NC(N->GroupStart());
        for (const RowMove &m : send)
            for (int p = 0; p < P; ++p)
                NC(N->Send(f + p * plane + (size_t)m.y0 * w, (size_t)(m.y1 - m.y0) * w, ncclDouble, m.peer, pl->nccl_comm, st));
        for (const RowMove &m : recv)
            for (int p = 0; p < P; ++p)
                NC(N->Recv(f + p * plane + (size_t)m.y0 * w, (size_t)(m.y1 - m.y0) * w, ncclDouble, m.peer, pl->nccl_comm, st));
        NC(N->GroupEnd());
        return 0;
    }
    if (base == B200P_XCHG_GATHER_RC) {
        // `level` is the first replicated level: rank q restricted the halves of its rows of the level above
        const int h1 = L.info.height, up = pl->strip_levels - 1;
        auto rows = [&](int q, int &a, int &b) {
            const int *r = pl->ranges_all.data() + ((size_t)q * pl->strip_levels + up) * 6;
            a = r[0] / 2;
            b = q == nr - 1 ? h1 : r[1] / 2;
        };
        int a0, b0;
        rows(me, a0, b0);
        NC(N->GroupStart());
        for (int q = 0; q < nr; ++q) {
            if (q == me) continue;
            int a, b;
            rows(q, a, b);
            for (int p = 0; p < P; ++p) {
                NC(N->Send(f + p * plane + (size_t)a0 * w, (size_t)(b0 - a0) * w, ncclDouble, q, pl->nccl_comm, st));
                NC(N->Recv(f + p * plane + (size_t)a * w, (size_t)(b - a) * w, ncclDouble, q, pl->nccl_comm, st));
            }
        }
        NC(N->GroupEnd());
        return 0;
    }
    return fail_arg(B200P_ERR_ARG, "unknown exchange %d", base);
}

// kind = base + 16 * level of the field (include/b200paint.h)
static int strip_exchange(b200p_plan *pl, int kind, void *d_ptr, cudaStream_t st, int level = 0) {
    if (pl->nccl_comm) return strip_exchange_nccl(pl, kind, level, d_ptr, st);
    if (!pl->exchange) return fail_arg(B200P_ERR_STATE, "strip mode needs an exchange callback");
    kind += 16 * level;
    const int rc = pl->exchange(pl->exchange_user, kind, d_ptr, (void *)st);
    if (rc) return fail_arg(B200P_ERR_STATE, "strip exchange %d failed (%d)", kind, rc);
    return 0;
}

static bool rows4_ok(const LevelHost &L, const double *u, const double *b) {
    const size_t plane = (size_t)L.info.height * L.info.width;
    return L.info.width % 4 == 0 && L.info.width >= 8 && plane % 4 == 0 && ((uintptr_t)u % 16) == 0 &&
           ((uintptr_t)b % 16) == 0 && ((uintptr_t)L.d_mask % 4) == 0;
}

// rm (right-hand side = where(mask, known, 0)) is only used by the solve drivers, where the iterate equals
// `known` at mask pixels after every step (flat init, prolongate_solution, corrections that are exactly 0
// there): the row walkers then skip the b - u evaluation at mask pixels.  B200P_TRUST_MASK=0 evaluates it.
static bool trust_mask_enabled() {
    const char *e = getenv("B200P_TRUST_MASK");
    return !(e && *e == '0');
}

static RowsArgs rows_args(b200p_plan *pl, const LevelHost &L, const double *u, const double *b,
                          const int *pred) {
    RowsArgs R;
    R.u = u;
    R.b = b;
    R.mask = L.d_mask;
    R.h = L.info.height;
    R.w = L.info.width;
    R.hinv2 = L.dev.hinv2;
    R.channels = pl->C;
    R.plane = (size_t)L.info.height * L.info.width;
    R.pred = pred;
    R.rows_per_cta = rows_chunk(L.info.height);
    R.y_lo = L.own_lo;
    R.y_hi = L.own_hi;
    R.partial = pl->d_partial;
    R.partial_flag = pl->d_partial_flag;
    R.counter = pl->d_counter;
    R.rs_out = pl->d_rs;
    R.flag_out = pl->d_mflag;
    R.trust = 0;
    return R;
}

// ---- tensor maps (cuTensorMapEncodeTiled through the runtime's driver entry point: no libcuda link)
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

static EncodeTiledFn tensor_map_encoder() {
    static EncodeTiledFn fn = []() -> EncodeTiledFn {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        return (EncodeTiledFn)p;
    }();
    return fn;
}

// (P, h, w) planes of fp64 (elem = 8) or bytes (elem = 1) as a 3-D tensor; box = bw x bh x 1 elements.
static int encode_plane_map(CUtensorMap *tm, const void *base, int elem, int w, int h, int planes, int box_w, int box_h) {
    EncodeTiledFn enc = tensor_map_encoder();
    if (!enc) return fail_arg(B200P_ERR_STATE, "cuTensorMapEncodeTiled is not available in this driver");
    cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)w * elem, (cuuint64_t)w * h * elem};
    cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(tm, elem == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 3,
                     const_cast<void *>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail_arg(B200P_ERR_STATE, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return 0;
}

#if B200P_LAB
static int encode_field_map(CUtensorMap *tm, const double *base, int w, int h, int planes, int box_w, int box_h) {
    return encode_plane_map(tm, base, 8, w, h, planes, box_w, box_h);
}
#endif

// K4 / K5: fine rows of coarse rows [Ylo, Yhi) (strip mode passes a sub-range; the whole plane otherwise).  Whole planes
// whose rows are 16-byte multiples in every array go through the TMA tile pipeline (kernels_rows_tma.cuh).
template <bool SOLUTION>
static int launch_prolongate(const double *coarse, const uint8_t *fmask, const double *frhs, int h, int w, int channels,
                             int planes, const int *pred, double *u, int Ylo, int Yhi, cudaStream_t st) {
    const int hc = (h + 1) >> 1, wc = (w + 1) >> 1;
    static const int want_tma = getenv("B200P_PROLONG_TMA") ? atoi(getenv("B200P_PROLONG_TMA")) : 1;
    if (want_tma && Ylo == 0 && Yhi >= hc && w % 16 == 0 && w >= RT_W && h >= 4 * RT_R && planes % channels == 0 &&
        ((uintptr_t)fmask % 16) == 0 && ((uintptr_t)coarse % 16) == 0 && ((uintptr_t)u % 16) == 0) {
        ProlongArgs A{h, w, channels, 32 * RT_R, pred, frhs, u};
        CUtensorMap tc, tm, tu;
        int rc = encode_plane_map(&tc, coarse, 8, wc, hc, planes, PT_CW, PT_CR);
        if (!rc) rc = encode_plane_map(&tm, fmask, 1, w, h, planes / channels, RT_W, RT_R);
        if (!rc) rc = SOLUTION ? 0 : encode_plane_map(&tu, u, 8, w, h, planes, RT_W, RT_R);
        if (rc) return rc;
        if (SOLUTION) tu = tc;
        static bool attr = false;
        if (!attr) {
            CU(cudaFuncSetAttribute(prolongate_tma_kernel<SOLUTION>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)prolong_tma_smem(SOLUTION)));
            attr = true;
        }
        dim3 g((w + RT_W - 1) / RT_W * channels, (h + A.rows_per_cta - 1) / A.rows_per_cta, planes / channels);
        prolongate_tma_kernel<SOLUTION><<<g, PT_THREADS, prolong_tma_smem(SOLUTION), st>>>(A, tc, tm, tu);
    } else {
        prolongate_kernel<SOLUTION><<<grid2x(wc, min(Yhi, hc) - Ylo, planes), ST_THREADS, 0, st>>>(
            coarse, fmask, frhs, h, w, channels, pred, u, Ylo, Yhi);
    }
    CU(cudaGetLastError());
    return 0;
}

// K1: rs[p] = ||b - A u||^2, mflag[p].  UM/RM as in residual_px.
static int launch_norm(b200p_plan *pl, const LevelHost &L, const double *u, const double *b,
                       bool um, bool rm, const int *pred, cudaStream_t st) {
    const size_t plane = (size_t)L.info.height * L.info.width;
    dim3 grid(pl->norm_ctas, pl->P);
    LaunchScope sc(pl, st, KK_NORM, field_bytes(pl, L, rm ? 1.0 : 2.0, 1.0));
#define NORM_ARGS u, b, L.d_mask, L.info.height, L.info.width, L.dev.hinv2, pl->C, plane, pred, \
                  pl->d_partial, pl->d_partial_flag, pl->d_counter, pl->d_rs, pl->d_mflag
    static const bool want_flat = !(getenv("B200P_FLAT_NORM") && atoi(getenv("B200P_FLAT_NORM")) == 0);
    if (want_flat && um && rm && u == b && L.info.width % 8 == 0 && ((uintptr_t)L.d_mask % 8) == 0) {
        // the flat initialisation's norm: work only next to mask pixels (kernels_rows.cuh, K1f)
        RowsArgs R = rows_args(pl, L, u, b, pred);
        dim3 g((L.info.width / 8 + FLAT_THREADS - 1) / FLAT_THREADS, (R.y_hi - R.y_lo + FLAT_ROWS - 1) / FLAT_ROWS, pl->F);
        flat_init_sqnorm_kernel<<<g, FLAT_THREADS, 0, st>>>(R);
        CU(cudaGetLastError());
        if (striped(pl, L)) {
            int rc2 = strip_exchange(pl, B200P_XCHG_SUM_RS, pl->d_rs, st);
            if (!rc2) rc2 = strip_exchange(pl, B200P_XCHG_MAX_FLAGS, pl->d_mflag, st);
            return rc2;
        }
        return 0;
    }
    static const bool want_tma = !(getenv("B200P_ROWS_TMA") && atoi(getenv("B200P_ROWS_TMA")) == 0);
    if (want_tma && !um && rows4_ok(L, u, b) && L.info.width % 16 == 0 && L.info.width >= RT_W &&
        L.info.height >= 4 * RT_R && ((uintptr_t)L.d_mask % 16) == 0) {
        // TMA-fed tile pipeline (kernels_rows_tma.cuh): bytes in flight independent of registers
        RowsArgs R = rows_args(pl, L, u, b, pred);
        R.trust = rm && trust_mask_enabled();
        const bool with_b = !(rm && R.trust);
        {
            // long strips amortise the pipeline fill (one DRAM latency per CTA); at least ~4 CTAs per SM slot overall
            static const int tiles = getenv("B200P_ROWS_TMA_TILES") ? atoi(getenv("B200P_ROWS_TMA_TILES")) : 32;
            R.rows_per_cta = std::max(4, tiles) * RT_R;
        }
        CUtensorMap tu, tm, tb;
        int rc = encode_plane_map(&tu, u, 8, L.info.width, L.info.height, pl->P, RT_BOXW, RT_R + 2);
        if (!rc) rc = encode_plane_map(&tm, L.d_mask, 1, L.info.width, L.info.height, pl->F, RT_W, RT_R);
        if (!rc) rc = with_b ? encode_plane_map(&tb, b, 8, L.info.width, L.info.height, pl->P, RT_W, RT_R) : 0;
        if (rc) return rc;
        if (!with_b) tb = tu;
        static bool attr = false;
        if (!attr) {
            CU(cudaFuncSetAttribute(residual_sqnorm_tma_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows_tma_smem(false)));
            CU(cudaFuncSetAttribute(residual_sqnorm_tma_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows_tma_smem(true)));
            CU(cudaFuncSetAttribute(residual_sqnorm_tma_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows_tma_smem(true)));
            attr = true;
        }
        dim3 g((L.info.width + RT_W - 1) / RT_W * pl->C, (R.y_hi - R.y_lo + R.rows_per_cta - 1) / R.rows_per_cta, pl->F);
        if (rm && !with_b) residual_sqnorm_tma_kernel<true, false><<<g, RT_THREADS, rows_tma_smem(false), st>>>(R, tu, tm, tb);
        else if (rm) residual_sqnorm_tma_kernel<true, true><<<g, RT_THREADS, rows_tma_smem(true), st>>>(R, tu, tm, tb);
        else residual_sqnorm_tma_kernel<false, true><<<g, RT_THREADS, rows_tma_smem(true), st>>>(R, tu, tm, tb);
        CU(cudaGetLastError());
        if (striped(pl, L)) {
            int rc2 = strip_exchange(pl, B200P_XCHG_SUM_RS, pl->d_rs, st);
            if (!rc2) rc2 = strip_exchange(pl, B200P_XCHG_MAX_FLAGS, pl->d_mflag, st);
            return rc2;
        }
        return 0;
    }
    if (rows4_ok(L, u, b)) {
        // four columns per thread, 16-byte loads (kernels_rows.cuh)
        RowsArgs R = rows_args(pl, L, u, b, pred);
        R.trust = rm && trust_mask_enabled();
        dim3 g4((L.info.width / 4 + ROWS4_THREADS - 1) / ROWS4_THREADS,
                (R.y_hi - R.y_lo + R.rows_per_cta - 1) / R.rows_per_cta, pl->P);
        if (um && rm) residual_sqnorm_rows4_kernel<true, true><<<g4, ROWS4_THREADS, 0, st>>>(R);
        else if (um) residual_sqnorm_rows4_kernel<true, false><<<g4, ROWS4_THREADS, 0, st>>>(R);
        else if (rm) residual_sqnorm_rows4_kernel<false, true><<<g4, ROWS4_THREADS, 0, st>>>(R);
        else residual_sqnorm_rows4_kernel<false, false><<<g4, ROWS4_THREADS, 0, st>>>(R);
        CU(cudaGetLastError());
        if (striped(pl, L)) {
            // the strip's partial sums (and mask-residual flags) -> totals over all ranks
            int rc = strip_exchange(pl, B200P_XCHG_SUM_RS, pl->d_rs, st);
            if (!rc) rc = strip_exchange(pl, B200P_XCHG_MAX_FLAGS, pl->d_mflag, st);
            return rc;
        }
        return 0;
    }
    if (striped(pl, L)) return fail_arg(B200P_ERR_UNSUPPORTED, "strip mode needs the row-walker kernels (width % 4 == 0)");
    const bool vec_ok = L.info.width % 2 == 0 && L.info.width >= 4 && ((uintptr_t)u % 16) == 0 &&
                        ((uintptr_t)L.d_mask % 2) == 0 && (plane % 2) == 0;
    if (vec_ok) {
        // vector path: two columns per thread, one partial per (column strip, row chunk)
        dim3 g((L.info.width / 2 + ST_THREADS - 1) / ST_THREADS, (L.info.height + NORM_ROWS - 1) / NORM_ROWS, pl->P);
        if (um && rm) residual_sqnorm_rows2_kernel<true, true><<<g, ST_THREADS, 0, st>>>(NORM_ARGS);
        else if (um) residual_sqnorm_rows2_kernel<true, false><<<g, ST_THREADS, 0, st>>>(NORM_ARGS);
        else if (rm) residual_sqnorm_rows2_kernel<false, true><<<g, ST_THREADS, 0, st>>>(NORM_ARGS);
        else residual_sqnorm_rows2_kernel<false, false><<<g, ST_THREADS, 0, st>>>(NORM_ARGS);
    } else if (!um) {
        // scalar row-walking kernel (odd widths)
        dim3 g((L.info.width + ST_THREADS - 1) / ST_THREADS, (L.info.height + NORM_ROWS - 1) / NORM_ROWS, pl->P);
        if (rm) residual_sqnorm_rows_kernel<true><<<g, ST_THREADS, 0, st>>>(NORM_ARGS);
        else residual_sqnorm_rows_kernel<false><<<g, ST_THREADS, 0, st>>>(NORM_ARGS);
    } else if (rm) residual_sqnorm_kernel<true, true><<<grid, ST_THREADS, 0, st>>>(NORM_ARGS);
    else residual_sqnorm_kernel<true, false><<<grid, ST_THREADS, 0, st>>>(NORM_ARGS);
#undef NORM_ARGS
    CU(cudaGetLastError());
    return 0;
}

static int local_cap(const b200p_plan *pl, const LevelHost &L) {
    return pl->cfg.local_max_iters > 0 ? pl->cfg.local_max_iters
                                       : 4 * L.info.block_h * L.info.block_w;
}

// Who writes a pixel?  Per axis: the block slots that cover it with a NON-ZERO weight (the ramp of
// partition.py:137-154 starts at 0, so the outermost pixel of every cut side drops out).  Returns false when
// those slots are not consecutive (never the case for the reference's ramps; the caller then keeps the
// full combine).  flag[slot * extent + i]: bit 0 = non-zero weight, bit 1 = "direct": the pixel has a
// single writer and (align > 1) so has every pixel of its aligned group of `align` pixels.
static bool axis_writers(const std::vector<int> &starts, const std::vector<double> &wts, int extent, int dim, int align,
                         std::vector<int> &first, std::vector<int> &count, std::vector<uint8_t> &flag,
                         std::vector<int> &direct_px) {
    first.assign(dim, -1);
    count.assign(dim, 0);
    flag.assign(starts.size() * (size_t)extent, 0);
    for (size_t s = 0; s < starts.size(); ++s)
        for (int i = 0; i < extent; ++i) {
            if (wts[s * extent + i] == 0.0) continue;
            const int x = starts[s] + i;
            flag[s * extent + i] |= 1;
            if (count[x] == 0) first[x] = (int)s;
            else if (first[x] + count[x] != (int)s) return false;
            count[x] += 1;
        }
    direct_px.assign(dim, 0);
    for (int g0 = 0; g0 < dim; g0 += align) {
        bool single = true;
        for (int x = g0; x < std::min(dim, g0 + align); ++x) single = single && count[x] == 1;
        for (int x = g0; x < std::min(dim, g0 + align); ++x) direct_px[x] = single ? 1 : 0;
    }
    for (int x = 0; x < dim; ++x) {
        if (count[x] < 1) return false;   // partition of unity: somebody must write every pixel
        if (direct_px[x] && wts[(size_t)first[x] * extent + (x - starts[first[x]])] != 1.0) return false;
    }
    for (size_t s = 0; s < starts.size(); ++s)
        for (int i = 0; i < extent; ++i)
            if (direct_px[starts[s] + i]) flag[s * extent + i] |= 2;
    // the block solve decides per PAIR of pixels (even start) from the first pixel's flags
    if (align > 1)
        for (size_t s = 0; s < starts.size(); ++s) {
            if (starts[s] & 1) return false;
            for (int i = 0; i + 1 < extent; i += 2) {
                const uint8_t a = flag[s * extent + i], b = flag[s * extent + i + 1];
                if ((a & 2) != (b & 2) || ((a & 2) && (a & 1) != (b & 1))) return false;
            }
        }
    return true;
}

// Tile variants of K2 (block extent -> <TW,TH,NWARP>).
enum { TILE_GENERIC = 0, TILE_32_A = 1, TILE_16 = 2, TILE_8 = 3, TILE_32_B = 4, TILE_32_C = 5,
       TILE_32_S = 6, TILE_32_T = 7, TILE_32_U = 8, TILE_32_TMA = 9, TILE_32_L = 10, TILE_32_W = 11,
       TILE_32_WQ = 12 };

static int tile_for(int bw, int bh) {
    if (bw == 32 && bh == 32) {
#if B200P_LAB
        const char *e = getenv("B200P_TILE32");
        if (e && *e == 'A') return TILE_32_A;
        if (e && *e == 'C') return TILE_32_C;
        if (e && *e == 'S') return TILE_32_S;
        if (e && *e == 'T') return TILE_32_T;
        if (e && *e == 'U') return TILE_32_U;
        if (e && *e == 'M') return TILE_32_TMA;
        if (e && *e == 'B') return TILE_32_B;
        if (e && *e == 'L') return TILE_32_L;  // two-warp register tile with the lean prologue
        if (e && *e == 'Q') return TILE_32_WQ; // warp per block, v and q in tensor memory
#endif
        return TILE_32_W;  // warp per block, v in tensor memory; falls back to B where not eligible
    }
    if (bw == 16 && bh == 16) return TILE_16;
    if (bw == 8 && bh == 8) return TILE_8;
    return TILE_GENERIC;
}

template <int TW, int TH, int NWARP, int REGCAP = 255>
static void launch_tile(const SweepArgs &A, bool rm, dim3 grid, cudaStream_t st) {
    if (rm) oras_sweep_tile_kernel<TW, TH, NWARP, true, REGCAP><<<grid, NWARP * 32, 0, st>>>(A);
    else oras_sweep_tile_kernel<TW, TH, NWARP, false, REGCAP><<<grid, NWARP * 32, 0, st>>>(A);
}

#if B200P_LAB
template <int TW, int TH, int NWARP, bool SR>
static void launch_tile_s(const SweepArgs &A, bool rm, dim3 grid, cudaStream_t st) {
    if (rm) oras_sweep_tile_s_kernel<TW, TH, NWARP, true, SR><<<grid, NWARP * 32, 0, st>>>(A);
    else oras_sweep_tile_s_kernel<TW, TH, NWARP, false, SR><<<grid, NWARP * 32, 0, st>>>(A);
}

template <int TW, int TH, int NWARP>
static void launch_fused(const FusedArgs &A, bool rm, int grid, cudaStream_t st) {
    const size_t smem = sizeof(double) * 4 * TH * NWARP * FUSED_THREADS;  // u_old staging of one band chunk
    if (rm) oras_fused_sweep_kernel<TW, TH, NWARP, true><<<grid, FUSED_THREADS, smem, st>>>(A);
    else oras_fused_sweep_kernel<TW, TH, NWARP, false><<<grid, FUSED_THREADS, smem, st>>>(A);
}

template <int TW, int TH, int NWARP>
static int fused_occupancy() {
    int occ = 0;
    const size_t smem = sizeof(double) * 4 * TH * NWARP * FUSED_THREADS;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, oras_fused_sweep_kernel<TW, TH, NWARP, true>,
                                                      FUSED_THREADS, smem) != cudaSuccess)
        occ = 0;
    return occ;
}
#endif

static void fill_sweep_args(b200p_plan *pl, const LevelHost &L, const double *u, const double *b,
                            const int *pred, SweepArgs &A) {
    A.L = L.dev;
    A.u = u;
    A.b = b;
    A.mask = L.d_mask;
    A.channels = pl->C;
    A.plane = (size_t)L.info.height * L.info.width;
    A.pred = pred;
    A.rs = pl->d_rs;
    A.mflag = pl->d_mflag;
    A.eta = pl->cfg.eta;
    A.max_iters = local_cap(pl, L);
    A.scratch = pl->d_scratch;
}

#if !B200P_LAB
static int launch_sweep_fused(b200p_plan *, const LevelHost &, UBuf &, const double *, bool, const int *, int *,
                              cudaStream_t) {
    return fail_arg(B200P_ERR_UNSUPPORTED, "the fused sweep is an experiment: build with -DB200P_EXPERIMENTS");
}
#else
// K2F: fused solve + combine, u.cur -> u.alt, then swap.
static int launch_sweep_fused(b200p_plan *pl, const LevelHost &L, UBuf &u, const double *b, bool rm,
                              const int *pred, int *unit_counter, cudaStream_t st) {
    FusedArgs A;
    fill_sweep_args(pl, L, u.cur, b, pred, A.S);
    A.S.scratch = L.d_ring;
    A.u_new = u.alt;
    A.R = L.R;
    A.lag = L.lag;
    A.nsx = L.nsx;
    A.nc = L.nc;
    A.cw = L.cw;
    A.P = pl->P;
    A.items_per_problem = L.info.ny * (L.nsx + L.nc);
    const size_t rows = (size_t)pl->P * L.info.ny;
    A.work = pl->d_sched;
    A.row_done = pl->d_sched + 1;
    A.band_done = pl->d_sched + 1 + rows;
    A.band_first_row = L.d_band_first_row;
    A.row_last_band = L.d_row_last_band;
    A.unit_counter = unit_counter;
    A.stats = pl->d_stats;
    CU(cudaMemsetAsync(pl->d_sched, 0, sizeof(unsigned) * (1 + 2 * rows), st));
    const long long total = (long long)pl->P * A.items_per_problem;
    const int grid = (int)std::min<long long>(total, L.fused_grid);
    // sweep = read u_old (+ b) + mask, write u_new; the corrections stay in L2
    LaunchScope sc(pl, st, KK_SWEEP, field_bytes(pl, L, rm ? 2.0 : 3.0, 1.0));
    switch (L.fused_tile) {
        case TILE_32_A: launch_fused<4, 2, 4>(A, rm, grid, st); break;
        case TILE_32_B: launch_fused<4, 4, 2>(A, rm, grid, st); break;
        case TILE_16: launch_fused<2, 4, 1>(A, rm, grid, st); break;
        default: return fail_arg(B200P_ERR_STATE, "level is not eligible for the fused sweep");
    }
    CU(cudaGetLastError());
    std::swap(u.cur, u.alt);
    return 0;
}

// ---- K2T: TMA-fed persistent sweep kernel (kernels_oras_tma.cuh)
// Combine on arrival inside K2 (no K2b launch, tiles consumed from L2): opt-in with B200P_ARRIVAL=1.
// Parity-exact, but measured slower than K2 + K2b (193 vs 243 fps): the fence + arrival atomics + two
// batches of L2 reads add ~5 k cycles of pure latency to every block in a kernel that is bound by
// latency at 6 blocks per SM, whereas K2b hides the same reads behind full occupancy.
static bool arrival_fusion_enabled() {
    const char *e = getenv("B200P_ARRIVAL");  // read at plan creation (the plan then owns the tables)
    return e && e[0] == '1';
}

static int tma_regcap() {
    static const int cap = getenv("B200P_TMA_REGCAP") ? atoi(getenv("B200P_TMA_REGCAP")) : 168;
    return cap;
}

template <bool RM, int REGCAP>
static int tma_grid() {
    static int grid = 0;
    if (!grid) {
        int occ = 0, sms = 148, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(oras_sweep_tma_kernel<RM, REGCAP>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, oras_sweep_tma_kernel<RM, REGCAP>, KT_THREADS, 0) !=
                cudaSuccess || occ < 1)
            occ = 4;
        grid = sms * occ;
    }
    return grid;
}

template <bool RM, int REGCAP>
static void launch_tma_t(const SweepTmaArgs &A, const CUtensorMap &tu, const CUtensorMap &tb, cudaStream_t st) {
    const int grid = std::min(A.total_items, tma_grid<RM, REGCAP>());
    oras_sweep_tma_kernel<RM, REGCAP><<<grid, KT_THREADS, 0, st>>>(A, tu, tb);
}

static int launch_sweep_tma(b200p_plan *pl, const LevelHost &L, const SweepArgs &S, bool rm, cudaStream_t st) {
    SweepTmaArgs A;
    A.S = S;
    A.mtab = L.d_mtab;
    A.total_items = pl->P * L.nblocks;
    CUtensorMap tu, tb;
    int rc = encode_field_map(&tu, S.u, L.info.width, L.info.height, pl->P, KT_WIN_W, KT_WIN_H);
    if (rc) return rc;
    if (rm) tb = tu;
    else if ((rc = encode_field_map(&tb, S.b, L.info.width, L.info.height, pl->P, 32, 32))) return rc;
    const int cap = tma_regcap();
#define KT_LAUNCH(CAP)                                      \
    do {                                                    \
        if (rm) launch_tma_t<true, CAP>(A, tu, tb, st);     \
        else launch_tma_t<false, CAP>(A, tu, tb, st);       \
    } while (0)
    if (cap == 255) KT_LAUNCH(255);
    else if (cap == 160) KT_LAUNCH(160);
    else if (cap == 128) KT_LAUNCH(128);
    else KT_LAUNCH(168);
#undef KT_LAUNCH
    return 0;
}
#endif  // B200P_LAB

// the 32x32 fast paths gather with 16-byte loads from a packed mask table: even width and starts, aligned fields
static bool tma_eligible(const LevelHost &L, const double *u, const double *b, bool rm) {
    return L.d_mtabw && L.info.width % 2 == 0 && ((uintptr_t)u % 16) == 0 && (rm || ((uintptr_t)b % 16) == 0);
}

static int launch_warp_sweep(const WarpSweepArgs &WA, bool rm, bool qt, int grid, cudaStream_t st) {
    const size_t smem = kw_table_bytes(WA.P, WA.S.L.nx, WA.S.L.ny);  // a few KB (P <= a few hundred problems)
#if B200P_LAB
    if (WA.u_out) {   // band combine: single-writer pixels go straight to the partner iterate
        if (rm) oras_sweep_warp_kernel<true, false, true><<<grid, KW_THREADS, smem, st>>>(WA);
        else oras_sweep_warp_kernel<false, false, true><<<grid, KW_THREADS, smem, st>>>(WA);
        CU(cudaGetLastError());
        return 0;
    }
#endif
#if B200P_LAB
    if (qt) {   // q = A p parked in tensor memory as well (measured slower)
        if (rm) oras_sweep_warp_kernel<true, true><<<grid, KW_THREADS, smem, st>>>(WA);
        else oras_sweep_warp_kernel<false, true><<<grid, KW_THREADS, smem, st>>>(WA);
        CU(cudaGetLastError());
        return 0;
    }
#endif
    (void)qt;
    if (rm) oras_sweep_warp_kernel<true, false><<<grid, KW_THREADS, smem, st>>>(WA);
    else oras_sweep_warp_kernel<false, false><<<grid, KW_THREADS, smem, st>>>(WA);
    CU(cudaGetLastError());
    return 0;
}

// K2W is persistent: resident CTAs per SM (register-limited) x SMs.
static int warp_sweep_grid() {
    static int grid = 0;
    if (!grid) {
        int occ = 0, sms = 148, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, oras_sweep_warp_kernel<true, false>, KW_THREADS, 0) !=
                cudaSuccess || occ < 2)
            occ = 2;  // 2 x 128 threads x 256 registers = the whole register file (the query reports 1)
        const char *e = getenv("B200P_KW_CTAS");
        if (e && atoi(e) > 0) occ = atoi(e);
        grid = sms * occ;
    }
    return grid;
}

// K2 + K2b: one ORAS sweep (in place on u.cur) using rs/mflag from the preceding K1.
static int launch_sweep_split(b200p_plan *pl, const LevelHost &L, UBuf &ub, const double *b, bool rm,
                              const int *pred, int *unit_counter, int tile, cudaStream_t st) {
    double *u = ub.cur;
    SweepArgs A;
    fill_sweep_args(pl, L, u, b, pred, A);
    A.iy0 = L.iy_lo;
    const bool u_zero = pl->u_zero_now;   // set by enqueue_vcycle for the first sweep on a fresh correction
    pl->u_zero_now = false;
    if (u_zero && !(tile == TILE_32_W && tma_eligible(L, u, b, rm)))
        return fail_arg(B200P_ERR_STATE, "implicit zero iterate on a level without the warp-per-block kernel");
    A.u_zero = u_zero ? 1 : 0;
    dim3 grid(L.nblocks, pl->P);
    // band combine (experiment, B200P_BAND=1 in a -DB200P_EXPERIMENTS build): K2W updates the single-writer
    // pixels itself, the combine pass visits the overlap bands only, u.cur -> u.alt.  Not in strip mode, and
    // not for the sweep that carries the 8-bit egress (its full combine pass writes every pixel of the image).
    const bool band = L.band && tile == TILE_32_W && tma_eligible(L, u, b, rm) && !striped(pl, L) && !pl->egress_now &&
                      ub.alt && ub.alt != ub.cur && ((uintptr_t)ub.alt % 16) == 0;
    if (striped(pl, L) && !((tile == TILE_32_L || tile == TILE_32_W || tile == TILE_32_WQ) && tma_eligible(L, u, b, rm)))
        return fail_arg(B200P_ERR_UNSUPPORTED, "strip mode needs the 32x32 lean block-solve kernel");
    {
        // read u (+ b) + mask, write the weighted correction tiles
        LaunchScope sc(pl, st, KK_SWEEP_SPLIT, field_bytes(pl, L, rm ? 2.0 : 3.0, 1.0));
        if ((tile == TILE_32_TMA || tile == TILE_32_L || tile == TILE_32_W || tile == TILE_32_WQ) &&
            !tma_eligible(L, u, b, rm))
            tile = TILE_32_B;
        switch (tile) {
            case TILE_32_W:
            case TILE_32_WQ: {
                WarpSweepArgs WA;
                WA.S = A;
                WA.mtab = L.d_mtabw;
                WA.nrows = L.iy_hi - L.iy_lo;  // strip mode: only the block rows of this rank
                WA.items_per_problem = WA.nrows * L.info.nx;
                WA.total = pl->P * WA.items_per_problem;
                // runs of consecutive items per claim only where every warp still gets several runs
                static const unsigned chunk_max = getenv("B200P_KW_CHUNK") ? (unsigned)atoi(getenv("B200P_KW_CHUNK")) : KW_CHUNK_MAX;
                WA.chunk = (long long)WA.total >= 8ll * chunk_max * KW_WARPS * warp_sweep_grid() ? chunk_max : 1u;
                const int per_cta = KW_WARPS * (int)WA.chunk;
                const int g = std::min((WA.total + per_cta - 1) / per_cta, warp_sweep_grid());
                WA.P = pl->P;
                WA.claim = L.d_claim;
                WA.u_out = band ? ub.alt : nullptr;
                WA.xflag = L.d_xflag;
                WA.yflag = L.d_yflag;
                kw_magic((unsigned)WA.items_per_problem, WA.m_ipp, WA.k_ipp);
                kw_magic((unsigned)L.info.nx, WA.m_nx, WA.k_nx);
                if ((unsigned)WA.total >= (1u << 30))
                    return fail_arg(B200P_ERR_UNSUPPORTED, "too many block solves per launch for the K2W item decode");
                if (kw_table_bytes(WA.P, L.info.nx, L.info.ny) > 40 * 1024)
                    return fail_arg(B200P_ERR_UNSUPPORTED, "too many problems / blocks per axis for the K2W tables");
                int rc = launch_warp_sweep(WA, rm, tile == TILE_32_WQ, g, st);
                if (rc) return rc;
                break;
            }
#if B200P_LAB
            case TILE_32_L: {
                static const int cap = getenv("B200P_REGCAP") ? atoi(getenv("B200P_REGCAP")) : 168;
                dim3 g3(L.info.nx, L.iy_hi - L.iy_lo, pl->P);  // strip mode: only the block rows of this rank
                if (L.d_cell_cnt && !striped(pl, L) && ub.alt && ub.alt != ub.cur) {
                    // combine on arrival: u.cur -> u.alt inside K2, no K2b launch
                    FuseArgs Fz;
                    Fz.u_out = ub.alt;
                    Fz.cell_cnt = L.d_cell_cnt;
                    Fz.cell_need = L.d_cell_need;
                    Fz.lastx = L.d_lastx;
                    Fz.lasty = L.d_lasty;
                    Fz.unit_counter = unit_counter;
                    CU(cudaMemsetAsync(L.d_cell_cnt, 0, sizeof(unsigned) * (size_t)pl->P * L.nblocks, st));
                    if (rm) oras_sweep_lean_kernel<true, 168, true><<<g3, 64, 0, st>>>(A, L.d_mtab, Fz);
                    else oras_sweep_lean_kernel<false, 168, true><<<g3, 64, 0, st>>>(A, L.d_mtab, Fz);
                    CU(cudaGetLastError());
                    std::swap(ub.cur, ub.alt);
                    return 0;
                }
#define KL_LAUNCH(CAP)                                                                      \
    do {                                                                                    \
        if (rm) oras_sweep_lean_kernel<true, CAP><<<g3, 64, 0, st>>>(A, L.d_mtab);          \
        else oras_sweep_lean_kernel<false, CAP><<<g3, 64, 0, st>>>(A, L.d_mtab);            \
    } while (0)
                if (cap == 255) KL_LAUNCH(255);
                else if (cap == 160) KL_LAUNCH(160);
                else if (cap == 152) KL_LAUNCH(152);
                else if (cap == 144) KL_LAUNCH(144);
                else if (cap == 128) KL_LAUNCH(128);
                else KL_LAUNCH(168);
#undef KL_LAUNCH
                break;
            }
            case TILE_32_TMA: {
                int rc = launch_sweep_tma(pl, L, A, rm, st);
                if (rc) return rc;
                break;
            }
            case TILE_32_A: launch_tile<4, 2, 4>(A, rm, grid, st); break;
            case TILE_32_C: launch_tile<4, 1, 8>(A, rm, grid, st); break;
            case TILE_32_S: launch_tile_s<4, 4, 2, false>(A, rm, grid, st); break;
            case TILE_32_T: launch_tile_s<4, 4, 2, true>(A, rm, grid, st); break;
            case TILE_32_U: launch_tile_s<4, 2, 4, false>(A, rm, grid, st); break;
#endif
            // two warps per 32x32 block, 4x4 pixels per thread: levels the warp-per-block kernel cannot take
            // (odd width, unaligned fields)
            case TILE_32_B: launch_tile<4, 4, 2, 168>(A, rm, grid, st); break;
            case TILE_16: launch_tile<2, 4, 1>(A, rm, grid, st); break;
            case TILE_8: launch_tile<1, 2, 1>(A, rm, grid, st); break;
            default: {
                const size_t smem = smem_cg_bytes(L.info.block_w, L.info.block_h);
                if (rm) oras_sweep_generic_kernel<true, 0><<<grid, GEN_THREADS, smem, st>>>(A);
                else oras_sweep_generic_kernel<false, 0><<<grid, GEN_THREADS, smem, st>>>(A);
            }
        }
        CU(cudaGetLastError());
    }
#if B200P_LAB
    if (band) {
        BandTables T;
        T.nzxf = L.d_nzxf; T.nzxn = L.d_nzxn; T.nzyf = L.d_nzyf; T.nzyn = L.d_nzyn;
        T.tp = KW_TP; T.tsz = KW_TSZ;
        if (L.n_band_rows > 0) {
            // band rows, every column: up to 2 x 2 tiles per pixel
            T.rows = L.d_band_rows; T.nrows = L.n_band_rows; T.cols = nullptr; T.ncols = L.info.width;
            dim3 g((T.ncols + ST_THREADS_COMBINE - 1) / ST_THREADS_COMBINE, (T.nrows + COMBINE_ROWS - 1) / COMBINE_ROWS, pl->P);
            LaunchScope sc(pl, st, KK_COMBINE, field_bytes(pl, L, 3.0, 0.0));
            oras_combine_band_kernel<2><<<g, ST_THREADS_COMBINE, 0, st>>>(L.dev, T, pl->d_scratch, A.plane, pred, pl->d_rs,
                                                                         u, ub.alt, unit_counter);
            CU(cudaGetLastError());
        }
        if (L.n_core_rows > 0 && L.n_band_cols > 0) {
            // the other rows, band columns only: one row slot, up to 2 tiles per pixel
            T.rows = L.d_core_rows; T.nrows = L.n_core_rows; T.cols = L.d_band_cols; T.ncols = L.n_band_cols;
            dim3 g((T.ncols + ST_THREADS_COMBINE - 1) / ST_THREADS_COMBINE, (T.nrows + COMBINE_ROWS - 1) / COMBINE_ROWS, pl->P);
            LaunchScope sc(pl, st, KK_COMBINE, 0.0);
            oras_combine_band_kernel<1><<<g, ST_THREADS_COMBINE, 0, st>>>(L.dev, T, pl->d_scratch, A.plane, pred, pl->d_rs,
                                                                         u, ub.alt, L.n_band_rows > 0 ? nullptr : unit_counter);
            CU(cudaGetLastError());
        }
        {
            // problems the sweep skipped keep their iterate across the buffer swap
            const size_t plane2 = A.plane / 2;
            dim3 g((unsigned)std::min<size_t>((plane2 + ST_THREADS_COMBINE - 1) / ST_THREADS_COMBINE, 148), pl->P);
            LaunchScope sc(pl, st, KK_COMBINE, 0.0);
            copy_skipped_problems_kernel<<<g, ST_THREADS_COMBINE, 0, st>>>(
                plane2, pred, pl->d_rs, reinterpret_cast<const double2 *>(u), reinterpret_cast<double2 *>(ub.alt));
            CU(cudaGetLastError());
        }
        std::swap(ub.cur, ub.alt);
        return 0;
    }
#endif
    {
        dim3 g((L.info.width + ST_THREADS_COMBINE - 1) / ST_THREADS_COMBINE,
               (L.own_hi - L.own_lo + COMBINE_ROWS - 1) / COMBINE_ROWS, pl->P);
        // read corrections + u, write u
        LaunchScope sc(pl, st, KK_COMBINE, field_bytes(pl, L, 3.0, 0.0));
        uint8_t *eg = pl->egress_now;   // set by enqueue_smooth for the last post-smoothing sweep of level 0
        pl->egress_now = nullptr;
        if (eg) pl->egress_fused = true;
        oras_combine_kernel<<<g, ST_THREADS_COMBINE, 0, st>>>(L.dev, pl->d_scratch, A.plane, pred,
                                                              pl->d_rs, u, unit_counter, L.own_lo, L.own_hi,
                                                              eg, pl->C, u_zero ? 1 : 0);
        CU(cudaGetLastError());
    }
    // strip mode: the rows the neighbours' block solves and stencils read from this strip
    if (striped(pl, L)) return strip_exchange(pl, B200P_XCHG_HALO_U, u, st, level_of(pl, L));
    return 0;
}

// path: -1 plan default; 0 generic split; >0 a tile id (split); -2 fused
static int launch_sweep(b200p_plan *pl, const LevelHost &L, UBuf &u, const double *b, bool rm,
                        const int *pred, int *unit_counter, int path, cudaStream_t st) {
    if ((path == -1 && L.fused) || path == -2)
        return launch_sweep_fused(pl, L, u, b, rm, pred, unit_counter, st);
    return launch_sweep_split(pl, L, u, b, rm, pred, unit_counter, path >= 0 ? path : L.tile, st);
}

// _smooth (multigrid.py:264-279): `units` sweeps with stop_norm = 0.  When
// have_norm is set, rs/mflag already describe (u, b) and the first K1 is skipped.
static int enqueue_smooth(b200p_plan *pl, const LevelHost &L, UBuf &u, const double *b, bool rm,
                          int units, const int *pred, int *unit_counter, bool have_norm,
                          cudaStream_t st, bool carries_egress = false) {
    for (int i = 0; i < units; ++i) {
        if (!(have_norm && i == 0)) {
            int rc = launch_norm(pl, L, u.cur, b, false, rm, pred, st);
            if (rc) return rc;
        }
        // the last sweep of the finest level's post-smoothing leaves the iterate the V-cycle ends with:
        // its combine pass also writes the 8-bit image (split path only; anything else takes the tail pass)
        const bool split = !L.fused && !(L.d_cell_cnt && !striped(pl, L));
        pl->egress_now = (carries_egress && i == units - 1 && split && !striped(pl, L)) ? pl->egress : nullptr;
        int rc = launch_sweep(pl, L, u, b, rm, pred, unit_counter, -1, st);
        pl->egress_now = nullptr;
        if (rc) return rc;
    }
    return 0;
}

static int launch_coarse(b200p_plan *pl, const LevelHost &L, double *u, const double *b,
                         bool rhs_masked, int init_mode, double tol, int max_sweeps, const int *pred,
                         int *units_out, int accumulate, cudaStream_t st, double *rel_out = nullptr,
                         bool record_history = false) {
    CoarseArgs A;
    A.L = L.dev;
    A.u = u;
    A.b = b;
    A.mask = L.d_mask;
    A.channels = pl->C;
    A.pred = pred;
    A.tol = tol;
    A.max_sweeps = max_sweeps;
    A.eta = pl->cfg.eta;
    A.max_iters = local_cap(pl, L);
    A.rhs_masked = rhs_masked ? 1 : 0;
    A.init_mode = init_mode;
    A.units_out = units_out;
    A.units_accumulate = accumulate;
    A.rel_out = rel_out;
    A.hist = record_history ? pl->d_hist : nullptr;
    A.histlen = pl->d_histlen;
    A.hist_cap = pl->hist_cap;
    const size_t n = (size_t)L.info.block_w * L.info.block_h;
    const size_t smem = smem_cg_bytes(L.info.block_w, L.info.block_h) + 2 * n * sizeof(double);
    LaunchScope sc(pl, st, KK_COARSE, field_bytes(pl, L, 3.0, 1.0));
    coarse_solve_kernel<<<pl->P, GEN_THREADS, smem, st>>>(A);
    CU(cudaGetLastError());
    return 0;
}

static int launch_control(b200p_plan *pl, int stage, cudaStream_t st) {
    LaunchScope sc(pl, st, KK_CONTROL, 0.0);
    fmg_control_kernel<<<1, 128, 0, st>>>(
        pl->P, stage, pl->d_rs, pl->cfg.tol_rel, pl->cfg.v_cycles_max, pl->d_baseline, pl->d_denom,
        pl->d_rel, pl->d_hist, pl->d_histlen, pl->d_active, pl->d_cycles, pl->d_units, pl->d_any,
        pl->cond_capture ? 1 : 0, pl->cond, pl->hist_cap);
    CU(cudaGetLastError());
    return 0;
}

static int launch_set_int(b200p_plan *pl, int *p, int n, int v, cudaStream_t st) {
    LaunchScope sc(pl, st, KK_CONTROL, 0.0);
    set_int_kernel<<<(n + 127) / 128, 128, 0, st>>>(p, n, v);
    CU(cudaGetLastError());
    return 0;
}

// build_hierarchy's data half (multigrid.py:249-260).
static int pack_masks(b200p_plan *pl, const LevelHost &L, cudaStream_t st) {
    if (!L.d_mtabw) return 0;
    LaunchScope sc(pl, st, KK_DOWN_MASK, (double)pl->F * L.nblocks * (32.0 * 32.0 + 4.0 * 32));
#if B200P_LAB
    pack_block_masks_kernel<<<dim3(L.nblocks, pl->F), KT_THREADS, 0, st>>>(
        L.dev, L.d_mask, (size_t)L.info.height * L.info.width, L.d_mtab, 0);
    CU(cudaGetLastError());
#endif
    pack_block_masks_warp_kernel<<<dim3((L.nblocks + KW_WARPS - 1) / KW_WARPS, pl->F), KW_THREADS, 0, st>>>(
        L.dev, L.d_mask, (size_t)L.info.height * L.info.width, L.d_mtabw);
    CU(cudaGetLastError());
    return 0;
}

static int enqueue_hierarchy(b200p_plan *pl, cudaStream_t st) {
    const int nl = (int)pl->lev.size();
    {
        int rc = pack_masks(pl, pl->lev[0], st);
        if (rc) return rc;
    }
    for (int l = 0; l + 1 < nl; ++l) {
        const LevelHost &f = pl->lev[l];
        LevelHost &c = pl->lev[l + 1];
        const int h = f.info.height, w = f.info.width;
        {
            LaunchScope sc(pl, st, KK_DOWN_MASK, 1.25 * pl->F * (double)h * w);
            if (words8_ok(w, f.d_mask, c.d_mask))
                downsample_mask8_kernel<<<grid2x(c.info.width / 8, c.info.height, pl->F), ST_THREADS, 0, st>>>(f.d_mask, h, w, c.d_mask);
            else
                downsample_mask_kernel<<<grid2x(c.info.width, c.info.height, pl->F), ST_THREADS, 0, st>>>(f.d_mask, h, w, c.d_mask);
            CU(cudaGetLastError());
        }
        {
            int rc = pack_masks(pl, c, st);
            if (rc) return rc;
        }
        {
            LaunchScope sc(pl, st, KK_DOWN_VALUES, field_bytes(pl, f, 1.25, 1.25));
            downsample_values_kernel<<<grid2x(c.info.width, c.info.height, pl->F), ST_THREADS, 0, st>>>(
                f.d_mask, c.d_mask, f.d_rhs, h, w, pl->C, pl->cfg.value_downsampling, c.d_rhs);
            CU(cudaGetLastError());
        }
    }
    return 0;
}

static UBuf level_ubuf(b200p_plan *pl, int level, double *d_u0) {
    LevelHost &L = pl->lev[level];
    UBuf u;
    u.cur = level == 0 ? d_u0 : L.d_u;
    u.alt = L.d_u_alt;
    return u;
}

// Brings the iterate back into `home` if an odd number of fused sweeps left it in the partner.
static int settle(b200p_plan *pl, const LevelHost &L, UBuf &u, double *home, cudaStream_t st) {
    if (u.cur == home) return 0;
    const size_t bytes = sizeof(double) * (size_t)pl->P * L.info.height * L.info.width;
    CU(cudaMemcpyAsync(home, u.cur, bytes, cudaMemcpyDeviceToDevice, st));
    std::swap(u.cur, u.alt);
    return 0;
}

// _cascade(to_tol=False) (multigrid.py:389-422) into d_u0 (level-0 iterate).
static int enqueue_cascade(b200p_plan *pl, double *d_u0, cudaStream_t st) {
    const int nl = (int)pl->lev.size();
    const double tol = std::min(pl->cfg.coarse_tol, pl->cfg.tol_rel);
    LevelHost &co = pl->lev[nl - 1];
    if (nl == 1) {
        // single level: the coarse solve IS the finest level; its sweeps count as fine units
        return launch_coarse(pl, co, d_u0, co.d_rhs, true, 1, tol, pl->cfg.coarse_max_iters, nullptr,
                             pl->d_units, 1, st);
    }
    int rc = launch_coarse(pl, co, co.d_u, co.d_rhs, true, 1, tol, pl->cfg.coarse_max_iters,
                           nullptr, nullptr, 0, st);
    if (rc) return rc;
    const double *coarse_u = co.d_u;
    for (int l = nl - 2; l >= 0; --l) {
        NvtxScope nv("cascade", l);
        LevelHost &f = pl->lev[l];
        const LevelHost &c = pl->lev[l + 1];
        UBuf uf = level_ubuf(pl, l, d_u0);
        {
            LaunchScope sc(pl, st, KK_PROLONG_SOL, field_bytes(pl, f, 1.25, 1.0));
            // strip mode: the coarse level is replicated, so the strip and its halo rows are
            // prolongated locally (no exchange)
            const int Ylo = f.ext_lo >> 1, Yhi = (f.ext_hi + 1) >> 1;
            if ((rc = launch_prolongate<true>(coarse_u, f.d_mask, f.d_rhs, f.info.height, f.info.width, pl->C, pl->P, nullptr,
                                              uf.cur, Ylo, Yhi, st)))
                return rc;
        }
        if (l > 0) {
            rc = enqueue_smooth(pl, f, uf, f.d_rhs, true, 1, nullptr, nullptr, false, st);
            if (rc) return rc;
        }
        coarse_u = uf.cur;
    }
    return 0;
}

// v_cycle (multigrid.py:335-371).  rm: b is read masked (level-0 `known` /
// hierarchy values); have_norm: rs/mflag are current for (u, b) on entry.
// The iterate enters and leaves in u.cur == its home buffer.
static int enqueue_vcycle(b200p_plan *pl, int level, UBuf &u, const double *b, bool rm,
                          const int *pred, int *unit_counter, bool have_norm, cudaStream_t st,
                          bool settle_home = true, bool u_is_zero = false) {
    const int nl = (int)pl->lev.size();
    LevelHost &L = pl->lev[level];
    const b200p_config &cfg = pl->cfg;
    int *uc = level == 0 ? unit_counter : nullptr;
    double *home = u.cur;
    if (level == nl - 1) {
        // single-level cycle: nu_pre + nu_post sweeps (always a single block here)
        return launch_coarse(pl, L, u.cur, b, rm, 2, 0.0, cfg.nu_pre + cfg.nu_post, pred, uc, 1, st);
    }
    int rc;
    {
        NvtxScope nv("vcycle pre-smooth", level);
        pl->u_zero_now = u_is_zero;   // the first sweep neither reads u nor needs it zeroed beforehand
        rc = enqueue_smooth(pl, L, u, b, rm, cfg.nu_pre, pred, uc, have_norm, st);
        pl->u_zero_now = false;
    }
    if (rc) return rc;
    LevelHost &Cc = pl->lev[level + 1];
    UBuf e = level_ubuf(pl, level + 1, nullptr);
    bool coarse_norm = false;  // K3 also produced ||r_c||^2 = residual norm^2 of the coarse system at e = 0
    bool e_implicit = false;   // the coarse correction starts as an implicit zero field
    {
        LaunchScope sc(pl, st, KK_RESTRICT, field_bytes(pl, L, rm ? 1.25 : 2.25, 1.25));
        // e is zeroed by the coarse solve (init_mode 0) on the coarsest level; on a level whose first sweep runs
        // the warp-per-block kernel it stays IMPLICITLY zero (that sweep does not read it, its combine pass
        // writes every pixel): no zeroing pass, no first read; everywhere else it is zeroed here
        const bool rows4 = rows4_ok(L, u.cur, b) && ((uintptr_t)Cc.d_rc % 16) == 0 && ((uintptr_t)Cc.d_mask % 2) == 0;
        static const bool want_implicit = !(getenv("B200P_IMPLICIT_ZERO") && atoi(getenv("B200P_IMPLICIT_ZERO")) == 0);
        e_implicit = want_implicit && level + 1 != nl - 1 && rows4 && !striped(pl, L) && !striped(pl, Cc) && cfg.nu_pre > 0 &&
                     !Cc.fused && Cc.tile == TILE_32_W && tma_eligible(Cc, e.cur, Cc.d_rc, false) && Cc.nblocks > 1;
        double *ez = (level + 1 == nl - 1 || e_implicit) ? nullptr : e.cur;
        if (rows4) {
            RestrictArgs RA;
            RA.R = rows_args(pl, L, u.cur, b, pred);
            RA.R.trust = rm && trust_mask_enabled();
            RA.cmask = Cc.d_mask;
            RA.rc = Cc.d_rc;
            RA.e_zero = ez;
            static const bool want_tma = !(getenv("B200P_ROWS_TMA") && atoi(getenv("B200P_ROWS_TMA")) != 1);   // 2: K1 only
            if (want_tma && L.info.width % 16 == 0 && L.info.width >= RT_W && L.info.height >= 4 * RT_R &&
                ((uintptr_t)L.d_mask % 16) == 0) {
                // TMA-fed tile pipeline (kernels_rows_tma.cuh)
                const bool with_b = !(rm && RA.R.trust);
                RA.R.rows_per_cta = 32 * RT_R;
                CUtensorMap tu, tm, tb;
                int rc2 = encode_plane_map(&tu, u.cur, 8, L.info.width, L.info.height, pl->P, RT_BOXW, RT_R + 2);
                if (!rc2) rc2 = encode_plane_map(&tm, L.d_mask, 1, L.info.width, L.info.height, pl->F, RT_W, RT_R);
                if (!rc2) rc2 = with_b ? encode_plane_map(&tb, b, 8, L.info.width, L.info.height, pl->P, RT_W, RT_R) : 0;
                if (rc2) return rc2;
                if (!with_b) tb = tu;
                static bool attr = false;
                if (!attr) {
                    CU(cudaFuncSetAttribute(residual_restrict_tma_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows_tma_smem(false)));
                    CU(cudaFuncSetAttribute(residual_restrict_tma_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows_tma_smem(true)));
                    CU(cudaFuncSetAttribute(residual_restrict_tma_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows_tma_smem(true)));
                    attr = true;
                }
                dim3 gt((L.info.width + RT_W - 1) / RT_W * pl->C, (RA.R.y_hi - RA.R.y_lo + RA.R.rows_per_cta - 1) / RA.R.rows_per_cta, pl->F);
                if (rm && !with_b) residual_restrict_tma_kernel<true, false><<<gt, RK_THREADS, rows_tma_smem(false), st>>>(RA, tu, tm, tb);
                else if (rm) residual_restrict_tma_kernel<true, true><<<gt, RK_THREADS, rows_tma_smem(true), st>>>(RA, tu, tm, tb);
                else residual_restrict_tma_kernel<false, true><<<gt, RK_THREADS, rows_tma_smem(true), st>>>(RA, tu, tm, tb);
            } else {
                dim3 g4((L.info.width / 4 + ROWS4_THREADS - 1) / ROWS4_THREADS,
                        (RA.R.y_hi - RA.R.y_lo + RA.R.rows_per_cta - 1) / RA.R.rows_per_cta, pl->P);
                if (rm) residual_restrict_rows4_kernel<true><<<g4, ROWS4_THREADS, 0, st>>>(RA);
                else residual_restrict_rows4_kernel<false><<<g4, ROWS4_THREADS, 0, st>>>(RA);
            }
            coarse_norm = !striped(pl, L);  // a strip only has its share of ||r_c||^2: the coarse level takes its own norm
        } else if (striped(pl, L)) {
            return fail_arg(B200P_ERR_UNSUPPORTED, "strip mode needs the row-walker kernels (width % 4 == 0)");
        } else {
            dim3 g = grid2x(Cc.info.width, Cc.info.height, pl->P);
            if (rm)
                residual_restrict_kernel<true><<<g, ST_THREADS, 0, st>>>(
                    u.cur, b, L.d_mask, Cc.d_mask, L.info.height, L.info.width, L.dev.hinv2, pl->C, pred,
                    Cc.d_rc, ez);
            else
                residual_restrict_kernel<false><<<g, ST_THREADS, 0, st>>>(
                    u.cur, b, L.d_mask, Cc.d_mask, L.info.height, L.info.width, L.dev.hinv2, pl->C, pred,
                    Cc.d_rc, ez);
        }
        CU(cudaGetLastError());
    }
    if (striped(pl, L)) {
        // every rank restricted its own rows: the next level either is striped too (it needs the rows
        // of its boundary blocks from the neighbours) or is replicated (all-gather); and the whole
        // coarse correction is zeroed (K3 only zeroed this strip's rows)
        if ((rc = strip_exchange(pl, Cc.is_strip ? B200P_XCHG_HALO_RC : B200P_XCHG_GATHER_RC, Cc.d_rc, st, level + 1)))
            return rc;
        if (level + 1 != nl - 1)
            CU(cudaMemsetAsync(e.cur, 0, sizeof(double) * (size_t)pl->P * Cc.info.height * Cc.info.width, st));
    }
    if (level + 1 == nl - 1) {
        const double tol = std::min(cfg.coarse_tol, cfg.tol_rel);
        rc = launch_coarse(pl, Cc, e.cur, Cc.d_rc, false, 0, tol, cfg.coarse_max_iters, pred,
                           nullptr, 0, st);
    } else {
        rc = enqueue_vcycle(pl, level + 1, e, Cc.d_rc, false, pred, nullptr, coarse_norm, st, false,
                            e_implicit && coarse_norm);
    }
    if (rc) return rc;
    {
        LaunchScope sc(pl, st, KK_PROLONG_CORR, field_bytes(pl, L, 2.25, 1.0));
        // strip mode: e is replicated, the strip and its halo rows are corrected locally
        const int Ylo = L.ext_lo >> 1, Yhi = (L.ext_hi + 1) >> 1;
        if ((rc = launch_prolongate<false>(e.cur, L.d_mask, nullptr, L.info.height, L.info.width, pl->C, pl->P, pred, u.cur,
                                           Ylo, Yhi, st)))
            return rc;
    }
    {
        NvtxScope nv("vcycle post-smooth", level);
        if ((rc = enqueue_smooth(pl, L, u, b, rm, cfg.nu_post, pred, uc, false, st, level == 0 && settle_home)))
            return rc;
    }
    // inner levels may end in the partner buffer (the caller prolongates from e.cur); the level
    // handed in from outside must end where it started
    return settle_home ? settle(pl, L, u, home, st) : 0;
}

// ====================================================================== CG pipelines ====
// The paper's comparison pipelines "cg", "ml-cg", "mg-cg": the same multigrid
// driver with _cg_run (solvers.py:97-128) as smoother / coarse solver.  Eager launches; the
// host reads the gates every few CG steps.
constexpr int CG_CTAS = 592;  // CTAs per problem of the flat CG kernels (4 per SM)

static CgArgs cg_args(b200p_plan *pl, const LevelHost &L, double *u, const double *b) {
    CgArgs A;
    A.mask = L.d_mask;
    A.b = b;
    A.u = u;
    A.r = pl->cg_r;
    A.p = pl->cg_p;
    A.q = pl->cg_q;
    A.h = L.info.height;
    A.w = L.info.width;
    A.channels = pl->C;
    A.plane = (size_t)L.info.height * L.info.width;
    A.hinv2 = L.dev.hinv2;
    A.gate = pl->cgs.gate;
    A.alpha = pl->cgs.alpha;
    A.beta = pl->cgs.beta;
    A.partial = pl->d_partial;
    A.counter = pl->d_counter;
    A.sum_out = pl->cgs.sum;
    return A;
}

// _cg_run on level L for the problems selected by `pred`.  denom_mode / tol / stop_abs / record as in
// cg_after_init_kernel.  Steps per problem end up in cgs.steps, |r| / denom in d_rel.
static int cg_run(b200p_plan *pl, const LevelHost &L, double *u, const double *b, bool rm, int max_steps,
                  int denom_mode, double tol, double stop_abs, bool record, const int *pred, cudaStream_t st) {
    const int nb = (pl->P + 127) / 128;
    CgArgs A = cg_args(pl, L, u, b);
    CgState &S = pl->cgs;
    const int ctas = (int)std::min<size_t>(CG_CTAS, (A.plane + CG_THREADS - 1) / CG_THREADS);
    dim3 grid(ctas, pl->P);
    const double fb = 8.0 * pl->P * (double)A.plane;
    {
        LaunchScope sc(pl, st, KK_CONTROL, 0.0);
        cg_begin_kernel<<<nb, 128, 0, st>>>(pl->P, pred, S);
        CU(cudaGetLastError());
    }
    {
        LaunchScope sc(pl, st, KK_CG, 4.0 * fb);
        if (rm) cg_field_kernel<0, true><<<grid, CG_THREADS, 0, st>>>(A);
        else cg_field_kernel<0, false><<<grid, CG_THREADS, 0, st>>>(A);
        CU(cudaGetLastError());
    }
    {
        LaunchScope sc(pl, st, KK_CONTROL, 0.0);
        cg_after_init_kernel<<<nb, 128, 0, st>>>(pl->P, S, denom_mode, tol, stop_abs, record ? 1 : 0);
        CU(cudaGetLastError());
    }
    // on_step (solvers.py:120-121): with a step hook on a recording run, the host looks at the step counters
    // after every update and hands out the iterate while they advance
    const bool hook = record && pl->step_cb;
    std::vector<int> seen, now;
    if (hook) {
        seen.assign(pl->P, 0);
        now.assign(pl->P, 0);
    }
    const bool host_checks = max_steps > 16 && !hook;
    int done = 0;
    while (done < max_steps) {
        const int chunk = hook ? 1 : std::min(host_checks ? 8 : max_steps, max_steps - done);
        if (host_checks) {
            int rc = launch_set_int(pl, pl->d_any, 1, 0, st);
            if (rc) return rc;
        }
        for (int k = 0; k < chunk; ++k) {
            {
                LaunchScope sc(pl, st, KK_CG, 2.0 * fb);
                cg_field_kernel<1, false><<<grid, CG_THREADS, 0, st>>>(A);
            }
            {
                LaunchScope sc(pl, st, KK_CONTROL, 0.0);
                cg_after_apply_kernel<<<nb, 128, 0, st>>>(pl->P, S);
            }
            {
                LaunchScope sc(pl, st, KK_CG, 5.0 * fb);
                cg_field_kernel<2, false><<<grid, CG_THREADS, 0, st>>>(A);
            }
            {
                LaunchScope sc(pl, st, KK_CONTROL, 0.0);
                cg_after_update_kernel<<<nb, 128, 0, st>>>(pl->P, S, max_steps, record ? 1 : 0, denom_mode,
                                                          host_checks ? pl->d_any : nullptr);
            }
            if (hook) {
                CU(cudaMemcpyAsync(now.data(), S.steps, pl->P * sizeof(int), cudaMemcpyDeviceToHost, st));
                CU(cudaStreamSynchronize(st));
                bool advanced = false;
                for (int p = 0; p < pl->P; ++p) advanced = advanced || now[p] != seen[p];
                seen = now;
                if (!advanced) return 0;                       // every problem stopped (tolerance, breakdown)
                const int crc = pl->step_cb(pl->step_user, u, L.info.height, L.info.width);
                if (crc) return fail_arg(B200P_ERR_STATE, "step callback returned %d", crc);
            }
            {
                LaunchScope sc(pl, st, KK_CG, 3.0 * fb);
                cg_dir_kernel<<<grid, CG_THREADS, 0, st>>>(A);
            }
            CU(cudaGetLastError());
        }
        done += chunk;
        if (host_checks) {
            CU(cudaMemcpyAsync(pl->h_any, pl->d_any, sizeof(int), cudaMemcpyDeviceToHost, st));
            CU(cudaStreamSynchronize(st));
            if (!*pl->h_any) break;
        }
    }
    return 0;
}

// _smooth with the CG smoother (multigrid.py:278-279): units * smoother_cg_iters steps, stop_norm 0
static int cg_smooth(b200p_plan *pl, const LevelHost &L, double *u, const double *b, bool rm, int units,
                     const int *pred, int *unit_counter, cudaStream_t st) {
    if (units <= 0) return 0;
    const int k = pl->cfg.smoother_cg_iters;
    int rc = cg_run(pl, L, u, b, rm, units * k, 0, 0.0, 0.0, false, pred, st);
    if (rc) return rc;
    if (unit_counter) {
        LaunchScope sc(pl, st, KK_CONTROL, 0.0);
        cg_units_kernel<<<(pl->P + 127) / 128, 128, 0, st>>>(pl->P, pred, pl->cgs.steps, k, unit_counter);
        CU(cudaGetLastError());
    }
    return 0;
}

static int cg_restrict(b200p_plan *pl, const LevelHost &L, const LevelHost &Cc, const double *u, const double *b,
                       bool rm, const int *pred, double *ez, cudaStream_t st) {
    LaunchScope sc(pl, st, KK_RESTRICT, field_bytes(pl, L, rm ? 1.25 : 2.25, 1.25));
    dim3 g = grid2x(Cc.info.width, Cc.info.height, pl->P);
    if (rm)
        residual_restrict_kernel<true><<<g, ST_THREADS, 0, st>>>(u, b, L.d_mask, Cc.d_mask, L.info.height,
                                                                 L.info.width, L.dev.hinv2, pl->C, pred, Cc.d_rc, ez);
    else
        residual_restrict_kernel<false><<<g, ST_THREADS, 0, st>>>(u, b, L.d_mask, Cc.d_mask, L.info.height,
                                                                  L.info.width, L.dev.hinv2, pl->C, pred, Cc.d_rc, ez);
    CU(cudaGetLastError());
    return 0;
}

// v_cycle (multigrid.py:335-371) with the CG smoother, in place on u
static int cg_vcycle(b200p_plan *pl, int level, double *u, const double *b, bool rm, const int *pred,
                     int *unit_counter, cudaStream_t st) {
    const int nl = (int)pl->lev.size();
    const b200p_config &cfg = pl->cfg;
    LevelHost &L = pl->lev[level];
    int *uc = level == 0 ? unit_counter : nullptr;
    int rc;
    if (level == nl - 1) return cg_smooth(pl, L, u, b, rm, cfg.nu_pre + cfg.nu_post, pred, uc, st);
    if ((rc = cg_smooth(pl, L, u, b, rm, cfg.nu_pre, pred, uc, st))) return rc;
    LevelHost &Cc = pl->lev[level + 1];
    double *e = Cc.d_u;
    if ((rc = cg_restrict(pl, L, Cc, u, b, rm, pred, e, st))) return rc;  // also e = 0
    if (level + 1 == nl - 1) {
        const double tol = std::min(cfg.coarse_tol, cfg.tol_rel);
        rc = cg_run(pl, Cc, e, Cc.d_rc, false, cfg.coarse_max_iters, 1, tol, 0.0, false, pred, st);
    } else {
        rc = cg_vcycle(pl, level + 1, e, Cc.d_rc, false, pred, nullptr, st);
    }
    if (rc) return rc;
    {
        LaunchScope sc(pl, st, KK_PROLONG_CORR, field_bytes(pl, L, 2.25, 1.0));
        if ((rc = launch_prolongate<false>(e, L.d_mask, nullptr, L.info.height, L.info.width, pl->C, pl->P, pred, u, 0,
                                           1 << 30, st)))
            return rc;
    }
    return cg_smooth(pl, L, u, b, rm, cfg.nu_post, pred, uc, st);
}

static int launch_flat_init(b200p_plan *pl, const LevelHost &L, double *u, cudaStream_t st);

// fmg_solve / cg_solve with the CG smoother: mode 0 "mg-cg", 1 "ml-cg", 2 "cg" (single level)
static int run_cg_pipeline(b200p_plan *pl, double *d_out, cudaStream_t st) {
    const int nl = (int)pl->lev.size();
    const b200p_config &cfg = pl->cfg;
    LevelHost &L0 = pl->lev[0];
    const int nb = (pl->P + 127) / 128;
    int rc;
    if (cfg.mode != 2 && (rc = enqueue_hierarchy(pl, st))) return rc;
    if ((rc = launch_norm(pl, L0, L0.d_rhs, L0.d_rhs, true, true, nullptr, st))) return rc;
    if ((rc = launch_control(pl, 0, st))) return rc;  // baseline; units, cycles, histlen = 0; active = 1
    if (cfg.mode == 2) {
        // cg_solve (solvers.py:140-186): flat init, stop at tol_rel * ||r0||, history [1, rn / r0 ...]
        if ((rc = launch_flat_init(pl, L0, d_out, st))) return rc;
        if ((rc = cg_run(pl, L0, d_out, L0.d_rhs, true, cfg.max_outer_iters, 1, cfg.tol_rel, 0.0, true, nullptr, st)))
            return rc;
        LaunchScope sc(pl, st, KK_CONTROL, 0.0);
        ml_finish_kernel<<<nb, 128, 0, st>>>(pl->P, pl->cgs.steps, pl->d_cycles, pl->d_units, pl->d_active);
        CU(cudaGetLastError());
        return 0;
    }
    // ---- _cascade (multigrid.py:389-422)
    const double ctol = std::min(cfg.coarse_tol, cfg.tol_rel);
    LevelHost &co = pl->lev[nl - 1];
    double *cu = nl == 1 ? d_out : co.d_u;
    if ((rc = launch_flat_init(pl, co, cu, st))) return rc;
    if ((rc = cg_run(pl, co, cu, co.d_rhs, true, cfg.coarse_max_iters, 1, ctol, 0.0, nl == 1 && cfg.mode == 1,
                     nullptr, st)))
        return rc;
    if (nl == 1) {
        // single level: the coarse solve is the finest level; its steps count as fine units
        LaunchScope sc(pl, st, KK_CONTROL, 0.0);
        if (cfg.mode == 1) {
            ml_finish_kernel<<<nb, 128, 0, st>>>(pl->P, pl->cgs.steps, pl->d_cycles, pl->d_units, pl->d_active);
        } else {
            cg_units_kernel<<<nb, 128, 0, st>>>(pl->P, nullptr, pl->cgs.steps, 1, pl->d_units);
        }
        CU(cudaGetLastError());
    }
    const double *coarse_u = cu;
    for (int l = nl - 2; l >= 0; --l) {
        LevelHost &f = pl->lev[l];
        const LevelHost &c = pl->lev[l + 1];
        double *uf = l == 0 ? d_out : f.d_u;
        {
            LaunchScope sc(pl, st, KK_PROLONG_SOL, field_bytes(pl, f, 1.25, 1.0));
            if ((rc = launch_prolongate<true>(coarse_u, f.d_mask, f.d_rhs, f.info.height, f.info.width, pl->C, pl->P, nullptr,
                                              uf, 0, 1 << 30, st)))
                return rc;
        }
        if (cfg.mode == 1) {
            // to_tol: denom = the level's flat-init defect (multigrid.py:413-417)
            if ((rc = launch_norm(pl, f, f.d_rhs, f.d_rhs, true, true, nullptr, st))) return rc;
            {
                LaunchScope sc(pl, st, KK_CONTROL, 0.0);
                ml_level_begin_kernel<<<nb, 128, 0, st>>>(pl->P, pl->d_rs, pl->cgs.denom, pl->d_gate, pl->d_sweeps);
                CU(cudaGetLastError());
            }
            if ((rc = cg_run(pl, f, uf, f.d_rhs, true, cfg.max_outer_iters, 2, cfg.tol_rel, 0.0, l == 0, nullptr, st)))
                return rc;
        } else if (l > 0) {
            if ((rc = cg_smooth(pl, f, uf, f.d_rhs, true, 1, nullptr, nullptr, st))) return rc;
        }
        coarse_u = uf;
    }
    if (cfg.mode == 1) {
        if (nl > 1) {
            LaunchScope sc(pl, st, KK_CONTROL, 0.0);
            ml_finish_kernel<<<nb, 128, 0, st>>>(pl->P, pl->cgs.steps, pl->d_cycles, pl->d_units, pl->d_active);
            CU(cudaGetLastError());
        }
        return 0;
    }
    // ---- V-cycles until converged (multigrid.py:466-481)
    if ((rc = launch_norm(pl, L0, d_out, L0.d_rhs, false, true, nullptr, st))) return rc;
    if ((rc = launch_control(pl, 1, st))) return rc;
    CU(cudaMemcpyAsync(pl->h_any, pl->d_any, sizeof(int), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    int done = 0;
    while (*pl->h_any && done < cfg.v_cycles_max) {
        if ((rc = cg_vcycle(pl, 0, d_out, L0.d_rhs, true, pl->d_active, pl->d_units, st))) return rc;
        if ((rc = launch_norm(pl, L0, d_out, L0.d_rhs, false, true, pl->d_active, st))) return rc;
        if ((rc = launch_control(pl, 2, st))) return rc;
        CU(cudaMemcpyAsync(pl->h_any, pl->d_any, sizeof(int), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        ++done;
    }
    return 0;
}

// _cascade(to_tol = False) with the CG smoother (multigrid.py:389-422), the stage form behind
// b200p_plan_cascade: coarsest level to min(coarse_tol, tol_rel), then prolongate + one smoothing unit per
// level (none on the finest).  No report state is touched.
static int cg_cascade_stage(b200p_plan *pl, double *d_out, cudaStream_t st) {
    const int nl = (int)pl->lev.size();
    const b200p_config &cfg = pl->cfg;
    const double ctol = std::min(cfg.coarse_tol, cfg.tol_rel);
    LevelHost &co = pl->lev[nl - 1];
    double *cu = nl == 1 ? d_out : co.d_u;
    int rc;
    if ((rc = launch_flat_init(pl, co, cu, st))) return rc;
    if ((rc = cg_run(pl, co, cu, co.d_rhs, true, cfg.coarse_max_iters, 1, ctol, 0.0, false, nullptr, st))) return rc;
    const double *coarse_u = cu;
    for (int l = nl - 2; l >= 0; --l) {
        LevelHost &f = pl->lev[l];
        double *uf = l == 0 ? d_out : f.d_u;
        {
            LaunchScope sc(pl, st, KK_PROLONG_SOL, field_bytes(pl, f, 1.25, 1.0));
            if ((rc = launch_prolongate<true>(coarse_u, f.d_mask, f.d_rhs, f.info.height, f.info.width, pl->C, pl->P,
                                              nullptr, uf, 0, 1 << 30, st)))
                return rc;
        }
        if (l > 0 && (rc = cg_smooth(pl, f, uf, f.d_rhs, true, 1, nullptr, nullptr, st))) return rc;
        coarse_u = uf;
    }
    return 0;
}

// _smooth_to_tol with the ORAS smoother on a multi-block level (multigrid.py:282-322): sweeps until
// ||r|| <= tol_rel * denom per problem, denom = the level's flat-init defect, at most max_outer_iters.
static int smooth_level_to_tol(b200p_plan *pl, LevelHost &f, UBuf &uf, bool record, cudaStream_t st) {
    const b200p_config &cfg = pl->cfg;
    const int nb = (pl->P + 127) / 128;
    int rc;
    // denom = ||b - A flat_init|| of this level (multigrid.py:413)
    if ((rc = launch_norm(pl, f, f.d_rhs, f.d_rhs, true, true, nullptr, st))) return rc;
    {
        LaunchScope sc(pl, st, KK_CONTROL, 0.0);
        ml_level_begin_kernel<<<nb, 128, 0, st>>>(pl->P, pl->d_rs, pl->d_denom, pl->d_gate, pl->d_sweeps);
        CU(cudaGetLastError());
    }
    int it = 0;
    for (;;) {
        const int chunk = 4;
        if ((rc = launch_set_int(pl, pl->d_any, 1, 0, st))) return rc;
        for (int k = 0; k < chunk && it <= cfg.max_outer_iters; ++k, ++it) {
            if ((rc = launch_norm(pl, f, uf.cur, f.d_rhs, false, true, pl->d_gate, st))) return rc;
            {
                LaunchScope sc(pl, st, KK_CONTROL, 0.0);
                ml_gate_kernel<<<nb, 128, 0, st>>>(pl->P, pl->d_rs, cfg.tol_rel, cfg.max_outer_iters,
                                                  pl->d_denom, pl->d_gate, pl->d_sweeps, pl->d_rel,
                                                  pl->d_hist, pl->d_histlen, record ? 1 : 0, pl->d_any,
                                                  pl->hist_cap);
                CU(cudaGetLastError());
            }
            if ((rc = launch_sweep(pl, f, uf, f.d_rhs, true, pl->d_gate, pl->d_sweeps, -1, st))) return rc;
        }
        CU(cudaMemcpyAsync(pl->h_any, pl->d_any, sizeof(int), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (!*pl->h_any || it > cfg.max_outer_iters) break;
    }
    return 0;
}

// oras_solve (solvers.py:427-485), the single-level "oras" pipeline: ORAS sweeps on the finest
// level from the flat initialisation until ||r|| <= tol_rel * ||r0||, at most max_outer_iters.
__global__ void flat_init_kernel(const uint8_t *__restrict__ mask, const double *__restrict__ known,
                                 size_t plane, int channels, size_t n, double *__restrict__ out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const size_t p = i / plane, px = i - p * plane;
    out[i] = mask[(p / channels) * plane + px] ? known[i] : 0.0;
}

static int launch_flat_init(b200p_plan *pl, const LevelHost &L, double *u, cudaStream_t st) {
    const size_t plane = (size_t)L.info.height * L.info.width, n = plane * pl->P;
    LaunchScope sc(pl, st, KK_CONVERT, 17.0 * n);
    flat_init_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(L.d_mask, L.d_rhs, plane, pl->C, n, u);
    CU(cudaGetLastError());
    return 0;
}

static int run_single_level(b200p_plan *pl, double *d_out, cudaStream_t st) {
    const int nl = (int)pl->lev.size();
    const b200p_config &cfg = pl->cfg;
    LevelHost &L0 = pl->lev[0];
    const int nb = (pl->P + 127) / 128;
    int rc;
    if ((rc = pack_masks(pl, L0, st))) return rc;
    if ((rc = launch_norm(pl, L0, L0.d_rhs, L0.d_rhs, true, true, nullptr, st))) return rc;
    if ((rc = launch_control(pl, 0, st))) return rc;  // baseline = ||b - A flat_init||
    if (nl == 1) {
        if ((rc = launch_coarse(pl, L0, d_out, L0.d_rhs, true, 1, cfg.tol_rel, cfg.max_outer_iters, nullptr,
                                pl->d_sweeps, 0, st, pl->d_rel, true)))
            return rc;
    } else {
        const size_t plane = (size_t)L0.info.height * L0.info.width, n = plane * pl->P;
        {
            LaunchScope sc(pl, st, KK_CONVERT, 17.0 * n);
            flat_init_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(L0.d_mask, L0.d_rhs, plane, pl->C, n, d_out);
            CU(cudaGetLastError());
        }
        UBuf uf = level_ubuf(pl, 0, d_out);
        if ((rc = smooth_level_to_tol(pl, L0, uf, true, st))) return rc;
        if ((rc = settle(pl, L0, uf, d_out, st))) return rc;
    }
    {
        LaunchScope sc(pl, st, KK_CONTROL, 0.0);
        ml_finish_kernel<<<nb, 128, 0, st>>>(pl->P, pl->d_sweeps, pl->d_cycles, pl->d_units, pl->d_active);
        CU(cudaGetLastError());
    }
    return 0;
}

// fmg_solve in "multilevel" mode (ml-oras; multigrid.py:449-464 with _cascade(to_tol=True),
// :389-418): coarsest level to min(coarse_tol, tol_rel); every finer level is initialised by
// prolongate_solution and smoothed until ||r|| <= tol_rel * (flat-init defect of that level),
// at most max_outer_iters sweeps.  A comparison pipeline of the paper, not the headline: it runs
// eagerly, the host reads the per-problem gates every few sweeps.
static int run_multilevel(b200p_plan *pl, double *d_out, cudaStream_t st) {
    const int nl = (int)pl->lev.size();
    const b200p_config &cfg = pl->cfg;
    LevelHost &L0 = pl->lev[0];
    const int nb = (pl->P + 127) / 128;
    int rc;
    if ((rc = enqueue_hierarchy(pl, st))) return rc;
    if ((rc = launch_norm(pl, L0, L0.d_rhs, L0.d_rhs, true, true, nullptr, st))) return rc;
    if ((rc = launch_control(pl, 0, st))) return rc;  // baseline; units, cycles, histlen = 0
    const double ctol = std::min(cfg.coarse_tol, cfg.tol_rel);
    LevelHost &co = pl->lev[nl - 1];
    if (nl == 1) {
        // single level: the coarse solve is the finest level (its per-evaluation history is not recorded)
        if ((rc = launch_coarse(pl, co, d_out, co.d_rhs, true, 1, ctol, cfg.coarse_max_iters, nullptr,
                                pl->d_sweeps, 0, st, pl->d_rel, true)))
            return rc;
    } else {
        if ((rc = launch_coarse(pl, co, co.d_u, co.d_rhs, true, 1, ctol, cfg.coarse_max_iters, nullptr,
                                nullptr, 0, st)))
            return rc;
        const double *coarse_u = co.d_u;
        for (int l = nl - 2; l >= 0; --l) {
            LevelHost &f = pl->lev[l];
            const LevelHost &c = pl->lev[l + 1];
            UBuf uf = level_ubuf(pl, l, d_out);
            double *home = uf.cur;
            {
                LaunchScope sc(pl, st, KK_PROLONG_SOL, field_bytes(pl, f, 1.25, 1.0));
                if ((rc = launch_prolongate<true>(coarse_u, f.d_mask, f.d_rhs, f.info.height, f.info.width, pl->C, pl->P,
                                                  nullptr, uf.cur, 0, 1 << 30, st)))
                    return rc;
            }
            if ((rc = smooth_level_to_tol(pl, f, uf, l == 0, st))) return rc;
            if ((rc = settle(pl, f, uf, home, st))) return rc;
            coarse_u = home;
        }
    }
    {
        LaunchScope sc(pl, st, KK_CONTROL, 0.0);
        ml_finish_kernel<<<nb, 128, 0, st>>>(pl->P, pl->d_sweeps, pl->d_cycles, pl->d_units, pl->d_active);
        CU(cudaGetLastError());
    }
    return 0;
}

// Front half of fmg_solve: hierarchy, baseline, cascade, first convergence check.
static int enqueue_front(b200p_plan *pl, double *d_out, cudaStream_t st) {
    LevelHost &L0 = pl->lev[0];
    int rc = enqueue_hierarchy(pl, st);
    if (rc) return rc;
    // baseline = ||b - A b|| with b = where(mask, known, 0) (multigrid.py:446)
    if ((rc = launch_norm(pl, L0, L0.d_rhs, L0.d_rhs, true, true, nullptr, st))) return rc;
    if ((rc = launch_control(pl, 0, st))) return rc;
    if ((rc = enqueue_cascade(pl, d_out, st))) return rc;
    if ((rc = launch_norm(pl, L0, d_out, L0.d_rhs, false, true, nullptr, st))) return rc;
    if ((rc = launch_control(pl, 1, st))) return rc;
    if (!pl->cond_capture) CU(cudaMemcpyAsync(pl->h_any, pl->d_any, sizeof(int), cudaMemcpyDeviceToHost, st));
    return 0;
}

// One V-cycle on level 0 + convergence check (multigrid.py:474-479).
static int enqueue_cycle(b200p_plan *pl, double *d_out, cudaStream_t st) {
    LevelHost &L0 = pl->lev[0];
    // rs/mflag are current on entry (the previous check's K1) iff nu_pre > 0 uses them first
    UBuf u = level_ubuf(pl, 0, d_out);
    int rc = enqueue_vcycle(pl, 0, u, L0.d_rhs, true, pl->d_active, pl->d_units,
                            (int)pl->lev.size() > 1, st);
    if (rc) return rc;
    if ((rc = launch_norm(pl, L0, d_out, L0.d_rhs, false, true, pl->d_active, st))) return rc;
    if ((rc = launch_control(pl, 2, st))) return rc;
    if (!pl->cond_capture) CU(cudaMemcpyAsync(pl->h_any, pl->d_any, sizeof(int), cudaMemcpyDeviceToHost, st));
    return 0;
}

template <class F>
static int run_graph(b200p_plan *pl, GraphSlot &slot, const void *k0, const void *k1, const void *k2,
                     cudaStream_t st, F &&enqueue) {
    if (!pl->cfg.use_graphs || pl->profiling) return enqueue(st);
    if (!slot.exec || slot.k0 != k0 || slot.k1 != k1 || slot.k2 != k2 || slot.k3 != pl->egress) {
        if (slot.exec) {
            cudaGraphExecDestroy(slot.exec);
            slot.exec = nullptr;
        }
        slot.kernels = 0;
        cudaGraph_t g = nullptr;
        CU(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        pl->launch_sink = &slot.kernels;
        int rc = enqueue(st);
        pl->launch_sink = nullptr;
        cudaError_t e = cudaStreamEndCapture(st, &g);
        if (rc) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        if (e != cudaSuccess) return fail_cuda(e, "cudaStreamEndCapture");
        e = cudaGraphInstantiate(&slot.exec, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return fail_cuda(e, "cudaGraphInstantiate");
        slot.k0 = k0;
        slot.k1 = k1;
        slot.k2 = k2;
        slot.k3 = pl->egress;
    }
    CU(cudaGraphLaunch(slot.exec, st));
    pl->launches += slot.kernels;
    return 0;
}

static void bind_level0(b200p_plan *pl, const uint8_t *d_mask, const double *d_known) {
    pl->lev[0].d_mask = const_cast<uint8_t *>(d_mask);
    pl->lev[0].d_rhs = const_cast<double *>(d_known);
}

static int set_smem_attrs() {
    static bool done = false;
    if (done) return 0;
    const int big = 227 * 1024;
    CU(cudaFuncSetAttribute(coarse_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(cudaFuncSetAttribute(oras_sweep_generic_kernel<true, 0>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(cudaFuncSetAttribute(oras_sweep_generic_kernel<false, 0>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(cudaFuncSetAttribute(oras_sweep_generic_kernel<false, 1>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, big));
#if B200P_LAB
    // K2S keeps CG state in static shared memory: ask for the large carve-out so that
    // 8 blocks per SM are resident
    const int carve = cudaSharedmemCarveoutMaxShared;
    CU(cudaFuncSetAttribute(oras_sweep_tile_s_kernel<4, 4, 2, true, false>, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    CU(cudaFuncSetAttribute(oras_sweep_tile_s_kernel<4, 4, 2, false, false>, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    CU(cudaFuncSetAttribute(oras_sweep_tile_s_kernel<4, 4, 2, true, true>, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    CU(cudaFuncSetAttribute(oras_sweep_tile_s_kernel<4, 4, 2, false, true>, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    CU(cudaFuncSetAttribute(oras_sweep_tile_s_kernel<4, 2, 4, true, false>, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    CU(cudaFuncSetAttribute(oras_sweep_tile_s_kernel<4, 2, 4, false, false>, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
#endif
    done = true;
    return 0;
}

// ================================================================ C-ABI =====
extern "C" {

const char *b200p_last_error(void) { return g_err.c_str(); }

int b200p_abi_version(void) { return B200P_ABI_VERSION; }

int b200p_has_experiments(void) { return B200P_LAB; }

int b200p_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int b200p_set_device(int device) {
    CU(cudaSetDevice(device));
    return 0;
}

int b200p_get_device(int *device) {
    if (!device) return fail_arg(B200P_ERR_ARG, "null argument");
    CU(cudaGetDevice(device));
    return 0;
}

void b200p_config_default(b200p_config *c, int width, int height, int channels) {
    memset(c, 0, sizeof *c);
    c->width = width;
    c->height = height;
    c->channels = channels;
    c->frames = 1;
    c->spacing = 1.0;
    c->block_size = 32;
    c->overlap = 6;
    c->nu_pre = 1;
    c->nu_post = 1;
    c->v_cycles_max = 100;
    c->value_downsampling = 1;
    c->coarse_tol = 1e-8;
    c->coarse_max_iters = 20000;
    c->tol_rel = 1e-3;
    c->alpha = 0.5;
    c->eta = 1e-5;
    c->local_max_iters = 0;
    c->use_graphs = 1;
    c->mode = 0;
    c->max_outer_iters = 10000;
    c->smoother = 0;
    c->smoother_cg_iters = 10;
}

int b200p_axis_starts(int dim, int block, int overlap, int64_t *out, int cap) {
    if (dim < 1) return fail_arg(B200P_ERR_ARG, "image dimensions must be >= 1, got %d", dim);
    if (overlap < 0 || block <= overlap)
        return fail_arg(B200P_ERR_ARG, "need block_size > overlap >= 0, got %d, %d", block, overlap);
    std::vector<int> s = axis_starts(dim, block, block - overlap);
    for (int i = 0; i < (int)s.size() && i < cap; ++i) out[i] = s[i];
    return (int)s.size();
}

int b200p_axis_weights(int dim, int block, int overlap, double *w, int cap) {
    if (dim < 1) return fail_arg(B200P_ERR_ARG, "image dimensions must be >= 1, got %d", dim);
    if (overlap < 0 || block <= overlap)
        return fail_arg(B200P_ERR_ARG, "need block_size > overlap >= 0, got %d, %d", block, overlap);
    std::vector<int> s = axis_starts(dim, block, block - overlap);
    const int bd = std::min(block, dim);
    std::vector<double> ww = axis_weights(s, bd, dim, overlap);
    for (int i = 0; i < (int)ww.size() && i < cap; ++i) w[i] = ww[i];
    return (int)ww.size();
}

int b200p_level_shapes(int width, int height, double spacing, int block, int overlap,
                       b200p_level_info *out, int cap) {
    if (width < 1 || height < 1)
        return fail_arg(B200P_ERR_ARG, "image dimensions must be >= 1, got %dx%d", width, height);
    if (overlap < 0 || block <= overlap)
        return fail_arg(B200P_ERR_ARG, "need block_size > overlap >= 0, got %d, %d", block, overlap);
    std::vector<b200p_level_info> v;
    level_shapes(width, height, spacing, block, overlap, v);
    for (int i = 0; i < (int)v.size() && i < cap; ++i) out[i] = v[i];
    return (int)v.size();
}

void b200p_plan_destroy(b200p_plan *pl) {
    if (!pl) return;
    prof_collect(pl);
    if (pl->d_stats) {
        unsigned long long h[8] = {0};
        cudaDeviceSynchronize();
        cudaMemcpy(h, pl->d_stats, 64, cudaMemcpyDeviceToHost);
        fprintf(stderr, "[b200p stats] solve: %llu items, %.0f cyc/item (+%.0f wait)  combine: %llu items, %.0f cyc/item (+%.0f wait)\n",
                h[4], h[4] ? (double)h[0] / h[4] : 0.0, h[4] ? (double)h[2] / h[4] : 0.0, h[5],
                h[5] ? (double)h[1] / h[5] : 0.0, h[5] ? (double)h[3] / h[5] : 0.0);
    }
    if (pl->g_front.exec) cudaGraphExecDestroy(pl->g_front.exec);
    if (pl->g_cycle.exec) cudaGraphExecDestroy(pl->g_cycle.exec);
    if (pl->g_solve.exec) cudaGraphExecDestroy(pl->g_solve.exec);
    if (pl->h_rep) cudaFreeHost(pl->h_rep);
    if (pl->aux_stream) cudaStreamDestroy(pl->aux_stream);
    for (void *p : pl->owned) cudaFree(p);
    if (pl->h_any) cudaFreeHost(pl->h_any);
    if (pl->h_pin) cudaFreeHost(pl->h_pin);
    if (pl->h_cnt) cudaFreeHost(pl->h_cnt);
    if (pl->d_cnt) cudaFree(pl->d_cnt);
    if (pl->h_sp_idx) cudaFreeHost(pl->h_sp_idx);
    if (pl->h_sp_val) cudaFreeHost(pl->h_sp_val);
    if (pl->d_sp_idx) cudaFree(pl->d_sp_idx);
    if (pl->d_sp_val) cudaFree(pl->d_sp_val);
    if (pl->own_stream) cudaStreamDestroy(pl->own_stream);
    delete pl;
}

int b200p_plan_create(const b200p_config *cfg, b200p_plan **out) {
    if (!cfg || !out) return fail_arg(B200P_ERR_ARG, "null argument");
    *out = nullptr;
    const b200p_config &c = *cfg;
    // same conditions as the reference's __post_init__ / build_partition checks
    if (c.width < 1 || c.height < 1)
        return fail_arg(B200P_ERR_ARG, "image dimensions must be >= 1, got %dx%d", c.width, c.height);
    if (c.channels < 1 || c.frames < 1)
        return fail_arg(B200P_ERR_ARG, "need channels >= 1 and frames >= 1");
    if (!(c.spacing > 0.0)) return fail_arg(B200P_ERR_ARG, "spacing must be positive, got %g", c.spacing);
    if (c.overlap < 0 || c.block_size <= c.overlap)
        return fail_arg(B200P_ERR_ARG, "need block_size > overlap >= 0, got %d, %d", c.block_size, c.overlap);
    if (c.block_size > B200P_MAX_BLOCK)
        return fail_arg(B200P_ERR_UNSUPPORTED, "block_size %d exceeds the supported maximum %d",
                        c.block_size, B200P_MAX_BLOCK);
    if (c.nu_pre < 0 || c.nu_post < 0 || c.nu_pre + c.nu_post < 1)
        return fail_arg(B200P_ERR_ARG, "need at least one smoothing iteration per cycle");
    if (!(c.tol_rel > 0.0 && c.tol_rel < 1.0))
        return fail_arg(B200P_ERR_ARG, "tol_rel must be in (0, 1), got %g", c.tol_rel);
    if (!(c.alpha > 0.0)) return fail_arg(B200P_ERR_ARG, "alpha must be positive, got %g", c.alpha);
    if (!(c.eta > 0.0)) return fail_arg(B200P_ERR_ARG, "local_tol_fraction must be positive, got %g", c.eta);
    if (c.value_downsampling != 0 && c.value_downsampling != 1)
        return fail_arg(B200P_ERR_ARG, "unknown value downsampling %d", c.value_downsampling);
    if (c.v_cycles_max < 0 || c.coarse_max_iters < 0 || c.local_max_iters < 0 || c.max_outer_iters < 0)
        return fail_arg(B200P_ERR_ARG, "iteration caps must be >= 0");
    if (c.mode < 0 || c.mode > 2) return fail_arg(B200P_ERR_ARG, "unknown mode %d", c.mode);
    if (c.smoother != 0 && c.smoother != 1) return fail_arg(B200P_ERR_ARG, "unknown smoother %d", c.smoother);
    if (c.smoother == 1 && c.smoother_cg_iters < 1)
        return fail_arg(B200P_ERR_ARG, "need at least one smoothing iteration per cycle");

    int ndev = 0;
    CU(cudaGetDeviceCount(&ndev));
    int rc = set_smem_attrs();
    if (rc) return rc;

    b200p_plan *pl = new b200p_plan();
    pl->cfg = c;
    pl->F = c.frames;
    pl->C = c.channels;
    pl->P = c.frames * c.channels;
    std::vector<b200p_level_info> shapes;
    level_shapes(c.width, c.height, c.spacing, c.block_size, c.overlap, shapes);
    if (std::max(shapes.back().height, shapes.back().width) > c.block_size) {
        delete pl;
        return fail_arg(B200P_ERR_UNSUPPORTED, "more than %d levels", B200P_MAX_LEVELS);
    }
    pl->lev.resize(shapes.size());
    const int stride = c.block_size - c.overlap;
    size_t scratch = 0;
#define PTRY(x)                      \
    do {                             \
        int r__ = (x);               \
        if (r__) {                   \
            b200p_plan_destroy(pl);  \
            return r__;              \
        }                            \
    } while (0)
    for (size_t l = 0; l < shapes.size(); ++l) {
        LevelHost &L = pl->lev[l];
        L.info = shapes[l];
        const int h = L.info.height, w = L.info.width;
        std::vector<int> xs = axis_starts(w, c.block_size, stride);
        std::vector<int> ys = axis_starts(h, c.block_size, stride);
        std::vector<double> wx = axis_weights(xs, L.info.block_w, w, c.overlap);
        std::vector<double> wy = axis_weights(ys, L.info.block_h, h, c.overlap);
        std::vector<int> cxf, cxn, cyf, cyn;
        axis_cover(xs, L.info.block_w, w, cxf, cxn);
        axis_cover(ys, L.info.block_h, h, cyf, cyn);
        L.nblocks = L.info.nx * L.info.ny;
        LevelDev &D = L.dev;
        D.h = h; D.w = w; D.nx = L.info.nx; D.ny = L.info.ny;
        D.bw = L.info.block_w; D.bh = L.info.block_h; D.nblocks = L.nblocks;
        D.spacing = L.info.spacing;
        D.hinv2 = 1.0 / (L.info.spacing * L.info.spacing);
        D.robin = c.alpha / L.info.spacing;
        D.g_in = 1.0 - D.robin / D.hinv2;
        PTRY(dev_upload(pl, xs, &D.xs));
        PTRY(dev_upload(pl, ys, &D.ys));
        PTRY(dev_upload(pl, wx, &D.wx));
        PTRY(dev_upload(pl, wy, &D.wy));
        PTRY(dev_upload(pl, cxf, &D.cxf));
        PTRY(dev_upload(pl, cxn, &D.cxn));
        PTRY(dev_upload(pl, cyf, &D.cyf));
        PTRY(dev_upload(pl, cyn, &D.cyn));
        L.tile = tile_for(D.bw, D.bh);
        L.own_lo = L.ext_lo = 0;
        L.own_hi = L.ext_hi = h;
        L.iy_lo = 0;
        L.iy_hi = L.info.ny;
        const size_t plane = (size_t)h * w;
#if B200P_LAB
        {
            const char *e = getenv("B200P_FUSED");
            const bool want = e && *e == '1';  // experimental; the split sweep (K2 + K2b) is faster
            const int ftile = (D.bw == 32 && D.bh == 32 && L.tile != TILE_32_A) ? TILE_32_B : L.tile;  // K2F knows A, B, 16
            const int bpc = ftile == TILE_32_A ? 1 : (ftile == TILE_32_B ? 2 : (ftile == TILE_16 ? 4 : 0));
            if (want && bpc > 0 && L.nblocks > 1) {
                L.fused = true;
                std::vector<int> first(L.info.ny), last(L.info.ny);
                int span = 0;
                for (int j = 0; j < L.info.ny; ++j) {
                    first[j] = cyf[ys[j]];
                    const int yl = ys[j] + D.bh - 1;
                    last[j] = cyf[yl] + cyn[yl] - 1;
                    span = std::max(span, last[j] - j);
                }
                const char *le = getenv("B200P_LAG");
                L.lag = le ? std::max(0, atoi(le)) : 8;
                const char *re = getenv("B200P_RING");
                L.R = L.lag + span + 1 + (re ? std::max(0, atoi(re)) : 24);
                L.nsx = (L.info.nx + bpc - 1) / bpc;
                L.cw = FUSED_THREADS;
                L.nc = (w + L.cw - 1) / L.cw;
                PTRY(dev_upload(pl, first, &L.d_band_first_row));
                PTRY(dev_upload(pl, last, &L.d_row_last_band));
                PTRY(dev_alloc(pl, &L.d_ring, (size_t)L.R * L.info.nx * D.bw * D.bh));
                PTRY(dev_alloc(pl, &L.d_u_alt, pl->P * plane));
                pl->sched_words = std::max(pl->sched_words, (size_t)1 + 2 * (size_t)pl->P * L.info.ny);
                int occ = 0, sms = 148;
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
                L.fused_tile = ftile;
                occ = ftile == TILE_32_A ? fused_occupancy<4, 2, 4>()
                      : (ftile == TILE_32_B ? fused_occupancy<4, 4, 2>() : fused_occupancy<2, 4, 1>());
                if (occ < 1) occ = 4;
                L.fused_grid = sms * occ;
            }
        }
#endif
        // the 32x32 fast path loads pixel pairs (16 bytes): even width and even block starts
        bool xs_even = true;
        for (int x : xs) xs_even = xs_even && (x % 2 == 0);
        if (D.bw == 32 && D.bh == 32 && w % 2 == 0 && xs_even)
        {
#if B200P_LAB
            PTRY(dev_alloc(pl, &L.d_mtab, (size_t)pl->F * L.nblocks * KT_THREADS));
#endif
            PTRY(dev_alloc(pl, &L.d_mtabw, (size_t)pl->F * L.nblocks * 32));
            PTRY(dev_alloc(pl, &L.d_claim, 4));
            CU(cudaMemset(L.d_claim, 0, 4 * sizeof(unsigned)));
            // band combine (experiment): single-writer pixels are updated by the block solve itself
            static const bool want_band = B200P_LAB && getenv("B200P_BAND") && atoi(getenv("B200P_BAND")) == 1;
            std::vector<int> nzxf, nzxn, nzyf, nzyn, dpx, dpy;
            std::vector<uint8_t> xflag, yflag;
            if (want_band && L.nblocks > 1 && (size_t)h * w >= 400000 &&   // small levels: one combine launch is cheaper
                axis_writers(xs, wx, D.bw, w, KW_ALIGN, nzxf, nzxn, xflag, dpx) &&
                axis_writers(ys, wy, D.bh, h, 1, nzyf, nzyn, yflag, dpy)) {
                std::vector<int> brows, crows, bcols;
                for (int y = 0; y < h; ++y) (dpy[y] ? crows : brows).push_back(y);
                for (int x = 0; x < w; ++x)
                    if (!dpx[x]) bcols.push_back(x);
                L.band = true;
                L.n_band_rows = (int)brows.size();
                L.n_core_rows = (int)crows.size();
                L.n_band_cols = (int)bcols.size();
                PTRY(dev_upload(pl, xflag, &L.d_xflag));
                PTRY(dev_upload(pl, yflag, &L.d_yflag));
                PTRY(dev_upload(pl, nzxf, &L.d_nzxf));
                PTRY(dev_upload(pl, nzxn, &L.d_nzxn));
                PTRY(dev_upload(pl, nzyf, &L.d_nzyf));
                PTRY(dev_upload(pl, nzyn, &L.d_nzyn));
                PTRY(dev_upload(pl, brows, &L.d_band_rows));
                PTRY(dev_upload(pl, crows, &L.d_core_rows));
                PTRY(dev_upload(pl, bcols, &L.d_band_cols));
                if (!L.d_u_alt) PTRY(dev_alloc(pl, &L.d_u_alt, (size_t)pl->P * h * w));
            }
        }
#if B200P_LAB
        if (L.d_mtab && L.nblocks > 1 && arrival_fusion_enabled()) {
            // cells = rectangles between consecutive block starts; a block overlaps the cells from its own
            // index to the last one starting inside its extent
            auto last_cell = [](const std::vector<int> &st, int extent) {
                std::vector<int> last(st.size());
                for (size_t i = 0; i < st.size(); ++i) {
                    size_t c = i;
                    while (c + 1 < st.size() && st[c + 1] < st[i] + extent) ++c;
                    last[i] = (int)c;
                }
                return last;
            };
            const std::vector<int> lastx = last_cell(xs, D.bw), lasty = last_cell(ys, D.bh);
            auto need_axis = [](const std::vector<int> &last) {
                std::vector<int> need(last.size(), 0);
                for (size_t i = 0; i < last.size(); ++i)
                    for (int c = (int)i; c <= last[i]; ++c) need[c] += 1;
                return need;
            };
            const std::vector<int> nxv = need_axis(lastx), nyv = need_axis(lasty);
            std::vector<int> need((size_t)L.nblocks);
            for (int cy = 0; cy < L.info.ny; ++cy)
                for (int cx = 0; cx < L.info.nx; ++cx) need[(size_t)cy * L.info.nx + cx] = nxv[cx] * nyv[cy];
            PTRY(dev_upload(pl, need, &L.d_cell_need));
            PTRY(dev_upload(pl, lastx, &L.d_lastx));
            PTRY(dev_upload(pl, lasty, &L.d_lasty));
            PTRY(dev_alloc(pl, &L.d_cell_cnt, (size_t)pl->P * L.nblocks));
            if (!L.d_u_alt) PTRY(dev_alloc(pl, &L.d_u_alt, (size_t)pl->P * h * w));
        }
#endif
        if (l > 0) {
            PTRY(dev_alloc(pl, &L.d_mask, pl->F * plane));
            PTRY(dev_alloc(pl, &L.d_rhs, pl->P * plane));
            PTRY(dev_alloc(pl, &L.d_u, pl->P * plane));
            PTRY(dev_alloc(pl, &L.d_rc, pl->P * plane));
        }
        if (L.nblocks > 1 || shapes.size() == 1)
            scratch = std::max(scratch, (size_t)pl->P * L.nblocks * (L.band ? (size_t)KW_TSZ : (size_t)D.bw * D.bh));
    }
    PTRY(dev_alloc(pl, &pl->d_scratch, scratch));
    PTRY(dev_alloc(pl, &pl->d_sched, std::max<size_t>(pl->sched_words, 4)));
    if (getenv("B200P_STATS")) {
        PTRY(dev_alloc(pl, &pl->d_stats, (size_t)8));
        CU(cudaMemset(pl->d_stats, 0, 64));
    }
    pl->norm_ctas = std::max(1, std::min(1024, (148 * 8 + pl->P - 1) / pl->P));
    size_t nparts = pl->norm_ctas;
    for (const LevelHost &L : pl->lev)
    {
        nparts = std::max(nparts, (size_t)((L.info.width + ST_THREADS - 1) / ST_THREADS) *
                                      ((L.info.height + NORM_ROWS - 1) / NORM_ROWS));
        nparts = std::max(nparts, (size_t)((L.info.width / 4 + ROWS4_THREADS - 1) / ROWS4_THREADS + 1) *
                                      ((L.info.height + 7) / 8));
    }
    if (c.smoother == 1) nparts = std::max(nparts, (size_t)CG_CTAS);
    PTRY(dev_alloc(pl, &pl->d_partial, (size_t)pl->P * nparts));
    PTRY(dev_alloc(pl, &pl->d_partial_flag, (size_t)pl->P * nparts));
    PTRY(dev_alloc(pl, &pl->d_counter, (size_t)pl->P));
    CU(cudaMemset(pl->d_counter, 0, sizeof(unsigned) * pl->P));
    PTRY(dev_alloc(pl, &pl->d_rs, (size_t)pl->P));
    PTRY(dev_alloc(pl, &pl->d_mflag, (size_t)pl->P));
    PTRY(dev_alloc(pl, &pl->d_active, (size_t)pl->P));
    PTRY(dev_alloc(pl, &pl->d_cycles, (size_t)pl->P));
    PTRY(dev_alloc(pl, &pl->d_units, (size_t)pl->P));
    PTRY(dev_alloc(pl, &pl->d_histlen, (size_t)pl->P));
    PTRY(dev_alloc(pl, &pl->d_any, (size_t)1));
    PTRY(dev_alloc(pl, &pl->d_baseline, (size_t)pl->P));
    PTRY(dev_alloc(pl, &pl->d_denom, (size_t)pl->P));
    PTRY(dev_alloc(pl, &pl->d_rel, (size_t)pl->P));
    {
        // every value the configured pipeline can record (SolveReport.history is never truncated in the
        // reference): V-cycles + 1 for mg-*, one per sweep / step (+ the start) for ml-* and the single-level
        // solvers, whose single-level hierarchies run under coarse_max_iters
        const b200p_config &hc = pl->cfg;
        long long need = (long long)hc.v_cycles_max + 2;
        if (hc.mode != 0) need = std::max(need, (long long)std::max(hc.max_outer_iters, hc.coarse_max_iters) + 2);
        pl->hist_cap = (int)std::min<long long>(std::max<long long>(need, B200P_MAX_HISTORY), 1 << 22);
    }
    PTRY(dev_alloc(pl, &pl->d_hist, (size_t)pl->P * pl->hist_cap));
    CU(cudaMemset(pl->d_hist, 0, sizeof(double) * (size_t)pl->P * pl->hist_cap));  // entries past histlen are copied out too
    PTRY(dev_alloc(pl, &pl->d_gate, (size_t)pl->P));
    PTRY(dev_alloc(pl, &pl->d_sweeps, (size_t)pl->P));
    PTRY(dev_alloc(pl, &pl->d_rn, (size_t)pl->P));
    if (c.smoother == 1) {
        const size_t n0 = (size_t)pl->P * c.width * c.height;
        PTRY(dev_alloc(pl, &pl->cg_r, n0));
        PTRY(dev_alloc(pl, &pl->cg_p, n0));
        PTRY(dev_alloc(pl, &pl->cg_q, n0));
        CgState &S = pl->cgs;
        PTRY(dev_alloc(pl, &S.rs, (size_t)pl->P));
        PTRY(dev_alloc(pl, &S.pq, (size_t)pl->P));
        PTRY(dev_alloc(pl, &S.alpha, (size_t)pl->P));
        PTRY(dev_alloc(pl, &S.beta, (size_t)pl->P));
        PTRY(dev_alloc(pl, &S.sum, (size_t)pl->P));
        PTRY(dev_alloc(pl, &S.stop, (size_t)pl->P));
        PTRY(dev_alloc(pl, &S.steps, (size_t)pl->P));
        PTRY(dev_alloc(pl, &S.denom, (size_t)pl->P));  // not d_denom: that is fmg_solve's own denominator
        S.rel = pl->d_rel;
        S.gate = pl->d_gate;
        S.hist = pl->d_hist;
        S.histlen = pl->d_histlen;
        S.hist_cap = pl->hist_cap;
    }
    {
        cudaError_t e = cudaMallocHost((void **)&pl->h_any, 64);
        if (e != cudaSuccess) {
            b200p_plan_destroy(pl);
            return fail_cuda(e, "cudaMallocHost");
        }
    }
#undef PTRY
    *out = pl;
    return 0;
}

int b200p_plan_num_levels(const b200p_plan *pl) { return pl ? (int)pl->lev.size() : 0; }

int b200p_plan_strip_ranges(const b200p_plan *pl, int levels, int rank, int nranks, int *out) {
    if (!pl || !out) return fail_arg(B200P_ERR_ARG, "null argument");
    return b200p_strip_ranges(pl->cfg.height, pl->cfg.block_size, pl->cfg.overlap, levels, rank, nranks, out);
}

int b200p_strip_ranges(int H, int block, int overlap, int levels, int rank, int nranks, int *out) {
    if (!out) return fail_arg(B200P_ERR_ARG, "null argument");
    if (H < 1 || block <= overlap || overlap < 0)
        return fail_arg(B200P_ERR_ARG, "need height >= 1 and block_size > overlap >= 0");
    if (levels < 1 || levels > 8) return fail_arg(B200P_ERR_ARG, "need 1 <= striped levels <= 8");
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return fail_arg(B200P_ERR_ARG, "bad rank %d of %d", rank, nranks);
    // strip boundaries on the finest level: even shares of the rows, rounded down to a multiple of
    // 2^levels so that they halve exactly on every striped level (2x2 cells never straddle a cut)
    const int q = 1 << levels;
    auto cut = [&](int k) { return k <= 0 ? 0 : (k >= nranks ? H : (int)(((long long)H * k / nranks) / q * q)); };
    const int a0 = cut(rank), b0 = cut(rank + 1);
    int h = H, need_lo = 0, need_hi = 0;  // rows of this level the finer level's prolongation reads
    for (int l = 0; l < levels; ++l) {
        const int own_lo = a0 >> l, own_hi = (rank + 1 == nranks) ? h : (b0 >> l);
        if (own_hi <= own_lo)
            return fail_arg(B200P_ERR_ARG, "empty strip on level %d for rank %d of %d (height %d)", l, rank, nranks, H);
        const std::vector<int> ys = axis_starts(h, block, block - overlap);
        const int ny = (int)ys.size(), bh = std::min(block, h);
        std::vector<int> cyf, cyn;
        axis_cover(ys, bh, h, cyf, cyn);
        // block rows that cover an owned pixel row are solved here (boundary rows redundantly by both sides)
        int iy_lo = ny, iy_hi = 0;
        for (int y = own_lo; y < own_hi; ++y) {
            iy_lo = std::min(iy_lo, cyf[y]);
            iy_hi = std::max(iy_hi, cyf[y] + cyn[y]);
        }
        // rows those block solves (1-pixel gather halo) and the stencils of the owned rows read, plus
        // what the finer level's prolongation onto ITS halo reads from this level
        int ext_lo = std::max(0, ys[iy_lo] - 1), ext_hi = std::min(h, ys[iy_hi - 1] + bh + 1);
        if (l > 0) {
            ext_lo = std::min(ext_lo, std::max(0, need_lo));
            ext_hi = std::max(ext_hi, std::min(h, need_hi));
        }
        ext_lo &= ~1;
        if (ext_hi < h) ext_hi = std::min(h, (ext_hi + 1) & ~1);
        int *o = out + 6 * l;
        o[0] = own_lo; o[1] = own_hi; o[2] = ext_lo; o[3] = ext_hi; o[4] = iy_lo; o[5] = iy_hi;
        need_lo = (ext_lo >> 1) - 1;
        need_hi = ((ext_hi + 1) >> 1) + 1;
        h = (h + 1) / 2;
    }
    return 0;
}

static void drop_graphs(b200p_plan *pl) {
    for (GraphSlot *g : {&pl->g_solve, &pl->g_front, &pl->g_cycle})
        if (g->exec) {
            cudaGraphExecDestroy(g->exec);
            g->exec = nullptr;
        }
}

static void leave_strip_mode(b200p_plan *pl) {
    pl->strip = false;
    pl->exchange = nullptr;
    pl->nccl_comm = nullptr;
    pl->ranges_all.clear();
    for (LevelHost &L : pl->lev) {
        L.is_strip = false;
        L.own_lo = L.ext_lo = 0; L.own_hi = L.ext_hi = L.info.height; L.iy_lo = 0; L.iy_hi = L.info.ny;
    }
    drop_graphs(pl);
}

static int enter_strip_mode(b200p_plan *pl, int levels, const int *r);

int b200p_plan_set_strip(b200p_plan *pl, int levels, const int *r, b200p_exchange_fn exchange, void *user) {
    if (!pl) return fail_arg(B200P_ERR_ARG, "null argument");
    if (pl->pending) return fail_arg(B200P_ERR_STATE, "a solve is pending on this plan");
    if (levels == 0 || !exchange) {  // back to the whole image
        if (levels != 0) return fail_arg(B200P_ERR_ARG, "strip mode needs an exchange callback");
        leave_strip_mode(pl);
        return 0;
    }
    if (!r) return fail_arg(B200P_ERR_ARG, "null argument");
    if (pl->cfg.use_graphs) return fail_arg(B200P_ERR_STATE, "strip plans with a host callback run eagerly: create the plan with use_graphs = 0");
    int rc = enter_strip_mode(pl, levels, r);
    if (rc) return rc;
    pl->nccl_comm = nullptr;
    pl->exchange = exchange;
    pl->exchange_user = user;
    return 0;
}

int b200p_plan_set_strip_nccl(b200p_plan *pl, int levels, const int *ranges_all, int rank, int nranks, void *comm) {
    if (!pl) return fail_arg(B200P_ERR_ARG, "null argument");
    if (pl->pending) return fail_arg(B200P_ERR_STATE, "a solve is pending on this plan");
    if (levels == 0) {
        leave_strip_mode(pl);
        return 0;
    }
    if (!ranges_all || !comm) return fail_arg(B200P_ERR_ARG, "null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail_arg(B200P_ERR_ARG, "bad rank %d of %d", rank, nranks);
    NcclApi *N = nccl_api();
    if (!N) return fail_arg(B200P_ERR_STATE, "libnccl.so.2 could not be loaded");
    int count = 0, urank = -1;
    NC(N->CommCount((ncclComm_t)comm, &count));
    NC(N->CommUserRank((ncclComm_t)comm, &urank));
    if (count != nranks || urank != rank)
        return fail_arg(B200P_ERR_ARG, "communicator is rank %d of %d, the strip layout says rank %d of %d", urank, count,
                        rank, nranks);
    int rc = enter_strip_mode(pl, levels, ranges_all + (size_t)rank * levels * 6);
    if (rc) return rc;
    pl->exchange = nullptr;
    pl->nccl_comm = (ncclComm_t)comm;
    pl->nccl_rank = rank;
    pl->nccl_nranks = nranks;
    pl->strip_levels = levels;
    pl->ranges_all.assign(ranges_all, ranges_all + (size_t)nranks * levels * 6);
    return 0;
}

int b200p_nccl_unique_id(void *id128) {
    NcclApi *N = nccl_api();
    if (!N) return fail_arg(B200P_ERR_STATE, "libnccl.so.2 could not be loaded");
    if (!id128) return fail_arg(B200P_ERR_ARG, "null argument");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    NC(N->GetUniqueId(static_cast<ncclUniqueId *>(id128)));
    return 0;
}

int b200p_nccl_comm_create(const void *id128, int rank, int nranks, void **comm) {
    NcclApi *N = nccl_api();
    if (!N) return fail_arg(B200P_ERR_STATE, "libnccl.so.2 could not be loaded");
    if (!id128 || !comm) return fail_arg(B200P_ERR_ARG, "null argument");
    ncclUniqueId id;
    memcpy(&id, id128, sizeof id);
    ncclComm_t c = nullptr;
    NC(N->CommInitRank(&c, nranks, id, rank));
    *comm = c;
    return 0;
}

int b200p_nccl_comm_destroy(void *comm) {
    NcclApi *N = nccl_api();
    if (!N) return fail_arg(B200P_ERR_STATE, "libnccl.so.2 could not be loaded");
    if (comm) NC(N->CommDestroy((ncclComm_t)comm));
    return 0;
}

int b200p_strip_halo_plan(const int *ranges_all, int levels, int level, int rank, int nranks, int *recv, int *send,
                          int cap) {
    if (!ranges_all || levels < 1 || level < 0 || level >= levels || nranks < 1 || rank < 0 || rank >= nranks)
        return fail_arg(B200P_ERR_ARG, "bad argument");
    std::vector<RowMove> r, s;
    halo_moves(ranges_all, levels, level, rank, nranks, r, s);
    const int n = (int)std::max(r.size(), s.size());
    if (recv && send)
        for (int i = 0; i < std::min(cap, n); ++i) {
            const RowMove none = {-1, 0, 0};
            const RowMove &a = i < (int)r.size() ? r[i] : none, &b = i < (int)s.size() ? s[i] : none;
            recv[3 * i] = a.peer; recv[3 * i + 1] = a.y0; recv[3 * i + 2] = a.y1;
            send[3 * i] = b.peer; send[3 * i + 1] = b.y0; send[3 * i + 2] = b.y1;
        }
    return n;
}

static int enter_strip_mode(b200p_plan *pl, int levels, const int *r) {
    if (pl->cfg.mode != 0 || pl->cfg.smoother != 0)
        return fail_arg(B200P_ERR_UNSUPPORTED, "strip mode covers the mg-oras path only");
    if (levels < 1 || levels + 1 > (int)pl->lev.size())
        return fail_arg(B200P_ERR_UNSUPPORTED, "need 1 <= striped levels < %d (the coarsest level stays replicated)",
                        (int)pl->lev.size());
    for (int l = 0; l < levels; ++l) {
        const LevelHost &L = pl->lev[l];
        const int H = L.info.height;
        const int *q = r + 6 * l;
        if (!L.d_mtabw || L.info.width % 4 != 0 || L.nblocks < 2)
            return fail_arg(B200P_ERR_UNSUPPORTED,
                            "strip mode needs 32x32 blocks with even starts and width %% 4 == 0 (level %d)", l);
        if (!(0 <= q[2] && q[2] <= q[0] && q[0] < q[1] && q[1] <= q[3] && q[3] <= H && 0 <= q[4] && q[4] < q[5] &&
              q[5] <= L.info.ny) || (q[0] & 1) || (q[2] & 1) || ((q[1] & 1) && q[1] != H) || ((q[3] & 1) && q[3] != H))
            return fail_arg(B200P_ERR_ARG, "inconsistent strip ranges on level %d", l);
    }
    for (int l = 0; l < (int)pl->lev.size(); ++l) {
        LevelHost &L = pl->lev[l];
        L.is_strip = l < levels;
        if (L.is_strip) {
            const int *q = r + 6 * l;
            L.own_lo = q[0]; L.own_hi = q[1]; L.ext_lo = q[2]; L.ext_hi = q[3]; L.iy_lo = q[4]; L.iy_hi = q[5];
        } else {
            L.own_lo = L.ext_lo = 0; L.own_hi = L.ext_hi = L.info.height; L.iy_lo = 0; L.iy_hi = L.info.ny;
        }
    }
    pl->strip = true;
    drop_graphs(pl);
    return 0;
}

int b200p_plan_level_rc(const b200p_plan *pl, int level, double **d_rc) {
    if (!pl || !d_rc || level < 1 || level >= (int)pl->lev.size()) return fail_arg(B200P_ERR_ARG, "bad level %d", level);
    *d_rc = pl->lev[level].d_rc;
    return 0;
}

int b200p_plan_level_info(const b200p_plan *pl, int level, b200p_level_info *out) {
    if (!pl || !out || level < 0 || level >= (int)pl->lev.size())
        return fail_arg(B200P_ERR_ARG, "bad level %d", level);
    *out = pl->lev[level].info;
    return 0;
}

int64_t b200p_plan_device_bytes(const b200p_plan *pl) { return pl ? pl->dev_bytes : 0; }
int64_t b200p_plan_launch_count(const b200p_plan *pl) { return pl ? pl->launches : 0; }

int b200p_plan_profile(b200p_plan *pl, int enable) {
    if (!pl) return fail_arg(B200P_ERR_ARG, "null plan");
    prof_collect(pl);
    pl->profiling = enable != 0;
    if (enable) {
        memset(pl->prof_ms, 0, sizeof pl->prof_ms);
        memset(pl->prof_bytes, 0, sizeof pl->prof_bytes);
        memset(pl->prof_launches, 0, sizeof pl->prof_launches);
    }
    return 0;
}

int b200p_plan_profile_kinds(void) { return KK_COUNT; }

const char *b200p_plan_profile_name(int kind) {
    return kind >= 0 && kind < KK_COUNT ? kKindNames[kind] : "";
}

int b200p_plan_profile_get(b200p_plan *pl, int kind, double *ms, int64_t *launches, double *bytes) {
    if (!pl || kind < 0 || kind >= KK_COUNT) return fail_arg(B200P_ERR_ARG, "bad kind %d", kind);
    prof_collect(pl);
    if (ms) *ms = pl->prof_ms[kind];
    if (launches) *launches = pl->prof_launches[kind];
    if (bytes) *bytes = pl->prof_bytes[kind];
    return 0;
}

static int ensure_report_block(b200p_plan *pl) {
    if (pl->h_rep) return 0;
    const size_t P = pl->P;
    const size_t bytes = P * (3 * sizeof(int) + 2 * sizeof(double)) + P * B200P_MAX_HISTORY * sizeof(double) + 64;
    CU(cudaHostAlloc(&pl->h_rep, bytes, cudaHostAllocMapped));
    memset(pl->h_rep, 0, bytes);
    // doubles first (alignment), then the ints
    double *d = reinterpret_cast<double *>(pl->h_rep);
    pl->rep.hist = d;
    pl->rep.baseline = d + P * B200P_MAX_HISTORY;
    pl->rep.rel = pl->rep.baseline + P;
    int *i = reinterpret_cast<int *>(pl->rep.rel + P);
    pl->rep.cycles = i;
    pl->rep.units = i + P;
    pl->rep.histlen = i + 2 * P;
    return 0;
}

// Device-side gather of the report fields into the mapped host record (no copy engine involved,
// so a lane's reports never queue behind another lane's bulk transfers).
static int enqueue_reports(b200p_plan *pl, cudaStream_t st) {
    int rc = ensure_report_block(pl);
    if (rc) return rc;
    if (pl->egress) {
        // 8-bit decode: problems whose image bytes no combine pass has written (no V-cycle needed, or a
        // pipeline / sweep variant without the fused egress) are converted here from the fp64 result
        const size_t plane = (size_t)pl->cfg.width * pl->cfg.height, npix = pl->F * plane;
        const int all = (pl->egress_fused && pl->cfg.mode == 0 && pl->cfg.smoother == 0) ? 0 : 1;
        LaunchScope sc(pl, st, KK_CONVERT, all ? 9.0 * pl->P * plane : 0.0);
        egress_u8_kernel<<<(unsigned)((npix + ST_THREADS - 1) / ST_THREADS), ST_THREADS, 0, st>>>(
            pl->egress_src, npix, pl->C, plane, pl->d_cycles, all, pl->egress);
        CU(cudaGetLastError());
    }
    LaunchScope sc(pl, st, KK_CONTROL, 0.0);
    const int n = pl->P * B200P_MAX_HISTORY;
    pack_reports_kernel<<<(n + 255) / 256, 256, 0, st>>>(pl->P, pl->d_cycles, pl->d_units, pl->d_histlen,
                                                        pl->d_baseline, pl->d_rel, pl->d_hist, pl->hist_cap, pl->rep);
    CU(cudaGetLastError());
    return 0;
}

static void read_reports(b200p_plan *pl, b200p_report *h_reports) {
    for (int p = 0; p < pl->P; ++p) {
        b200p_report &r = h_reports[p];
        memset(&r, 0, sizeof r);
        r.iterations = pl->rep.cycles[p];
        r.fine_smoother_iterations = pl->rep.units[p];
        r.history_len = pl->rep.histlen[p];
        r.final_rel_residual = pl->rep.rel[p];
        r.baseline_residual = pl->rep.baseline[p];
        r.init_residual = pl->rep.baseline[p];
        r.converged = pl->rep.rel[p] <= pl->cfg.tol_rel;
        memcpy(r.history, &pl->rep.hist[(size_t)p * B200P_MAX_HISTORY], sizeof(double) * B200P_MAX_HISTORY);
    }
}

// The whole of fmg_solve as ONE graph: front (hierarchy, baseline, cascade, first check) ->
// WHILE node whose body is one V-cycle + check (multigrid.py:474-479; the control kernel sets
// the loop condition on the device) -> report gather.  No host round trip inside a solve.
static int launch_solve_graph(b200p_plan *pl, const uint8_t *d_mask, const double *d_known, double *d_out,
                              cudaStream_t st) {
    GraphSlot &slot = pl->g_solve;
    if (!slot.exec || slot.k0 != d_mask || slot.k1 != d_known || slot.k2 != d_out || slot.k3 != pl->egress) {
        if (slot.exec) {
            cudaGraphExecDestroy(slot.exec);
            slot.exec = nullptr;
        }
        pl->egress_fused = false;
        int rc = ensure_report_block(pl);
        if (rc) return rc;
        if (!pl->aux_stream) CU(cudaStreamCreateWithFlags(&pl->aux_stream, cudaStreamNonBlocking));
        slot.kernels = 0;
        pl->cycle_kernels = 0;
        cudaGraph_t g = nullptr, body = nullptr, tmp = nullptr;
        cudaStreamCaptureStatus cs;
        const cudaGraphNode_t *deps = nullptr;
        size_t ndeps = 0;
        CU(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        pl->cond_capture = true;
        rc = 0;
        cudaError_t e = cudaStreamGetCaptureInfo_v2(st, &cs, nullptr, &g, &deps, &ndeps);
        if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&pl->cond, g, 0, cudaGraphCondAssignDefault);
        if (e == cudaSuccess) {
            pl->launch_sink = &slot.kernels;
            rc = enqueue_front(pl, d_out, st);
        }
        cudaGraphNode_t node = nullptr;
        if (e == cudaSuccess && !rc) e = cudaStreamGetCaptureInfo_v2(st, &cs, nullptr, &g, &deps, &ndeps);
        if (e == cudaSuccess && !rc) {
            cudaGraphNodeParams np = {};
            np.type = cudaGraphNodeTypeConditional;
            np.conditional.handle = pl->cond;
            np.conditional.type = cudaGraphCondTypeWhile;
            np.conditional.size = 1;
            e = cudaGraphAddNode(&node, g, deps, ndeps, &np);
            if (e == cudaSuccess) body = np.conditional.phGraph_out[0];
        }
        if (e == cudaSuccess && !rc)
            e = cudaStreamBeginCaptureToGraph(pl->aux_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
        if (e == cudaSuccess && !rc) {
            pl->launch_sink = &pl->cycle_kernels;
            rc = enqueue_cycle(pl, d_out, pl->aux_stream);
            cudaError_t e2 = cudaStreamEndCapture(pl->aux_stream, &tmp);
            if (e == cudaSuccess) e = e2;
        }
        if (e == cudaSuccess && !rc) e = cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies);
        if (e == cudaSuccess && !rc) {
            pl->launch_sink = &slot.kernels;
            rc = enqueue_reports(pl, st);
        }
        pl->launch_sink = nullptr;
        pl->cond_capture = false;
        cudaGraph_t full = nullptr;
        cudaError_t e3 = cudaStreamEndCapture(st, &full);
        if (rc) {
            if (full) cudaGraphDestroy(full);
            return rc;
        }
        if (e != cudaSuccess) {
            if (full) cudaGraphDestroy(full);
            return fail_cuda(e, "capture of the solve graph");
        }
        if (e3 != cudaSuccess) return fail_cuda(e3, "cudaStreamEndCapture");
        e = cudaGraphInstantiate(&slot.exec, full, 0);
        cudaGraphDestroy(full);
        if (e != cudaSuccess) return fail_cuda(e, "cudaGraphInstantiate");
        slot.k0 = d_mask;
        slot.k1 = d_known;
        slot.k2 = d_out;
        slot.k3 = pl->egress;
    }
    CU(cudaGraphLaunch(slot.exec, st));
    return 0;
}

static int solve_async_impl(b200p_plan *pl, const uint8_t *d_mask, const double *d_known, double *d_out,
                            uint8_t *d_egress, void *stream);

int b200p_solve_async(b200p_plan *pl, const uint8_t *d_mask, const double *d_known, double *d_out,
                      void *stream) {
    return solve_async_impl(pl, d_mask, d_known, d_out, nullptr, stream);
}

// d_egress: optional (F, h, w, C) 8-bit image the solve also leaves its result in (image_from_fields)
static int solve_async_impl(b200p_plan *pl, const uint8_t *d_mask, const double *d_known, double *d_out,
                            uint8_t *d_egress, void *stream) {
    if (!pl || !d_mask || !d_known || !d_out) return fail_arg(B200P_ERR_ARG, "null argument");
    if (pl->pending) return fail_arg(B200P_ERR_STATE, "a solve is pending on this plan: call b200p_solve_wait first");
    cudaStream_t st = (cudaStream_t)stream;
    const bool graphs = pl->cfg.use_graphs && !pl->profiling;
    pl->egress = d_egress;
    pl->egress_src = d_out;
    if (!graphs) pl->egress_fused = false;
    if (graphs && st == nullptr) {
        // stream capture is not allowed on the legacy default stream
        if (!pl->own_stream) CU(cudaStreamCreateWithFlags(&pl->own_stream, cudaStreamNonBlocking));
        CU(cudaDeviceSynchronize());
        st = pl->own_stream;
    }
    bind_level0(pl, d_mask, d_known);
    int rc;
    if (pl->cfg.mode != 0 || pl->cfg.smoother == 1) {
        if (pl->cfg.smoother == 1) rc = run_cg_pipeline(pl, d_out, st);
        else rc = pl->cfg.mode == 1 ? run_multilevel(pl, d_out, st) : run_single_level(pl, d_out, st);
        if (rc) return rc;
        pl->hierarchy_ready = true;
        if ((rc = enqueue_reports(pl, st))) return rc;
        pl->pending = true;
        pl->pending_stream = st;
        pl->pending_eager = true;
        return 0;
    }
    pl->pending_eager = !graphs;
    if (graphs && pl->strip && pl->nccl_comm && pl->nccl_warm) {
        // Strip mode with the library's own NCCL exchange: kernels and collectives of the front part and of
        // one V-cycle are two captured graphs; the host only reads the loop condition between replays.
        pl->pending_eager = true;
        if ((rc = run_graph(pl, pl->g_front, d_mask, d_known, d_out, st,
                            [&](cudaStream_t s) { return enqueue_front(pl, d_out, s); })))
            return rc;
        pl->hierarchy_ready = true;
        CU(cudaStreamSynchronize(st));
        int done = 0;
        while (*pl->h_any && done < pl->cfg.v_cycles_max) {
            if ((rc = run_graph(pl, pl->g_cycle, d_mask, d_known, d_out, st,
                                [&](cudaStream_t s) { return enqueue_cycle(pl, d_out, s); })))
                return rc;
            ++done;
            CU(cudaStreamSynchronize(st));
        }
        if ((rc = enqueue_reports(pl, st))) return rc;
    } else if (graphs && !pl->strip) {
        if ((rc = launch_solve_graph(pl, d_mask, d_known, d_out, st))) return rc;
        pl->hierarchy_ready = true;
    } else {
        pl->pending_eager = true;
        if (pl->strip && pl->nccl_comm) pl->nccl_warm = true;
        // eager: the host reads the loop condition after every cycle
        if ((rc = enqueue_front(pl, d_out, st))) return rc;
        pl->hierarchy_ready = true;
        CU(cudaStreamSynchronize(st));
        int done = 0;
        while (*pl->h_any && done < pl->cfg.v_cycles_max) {
            if ((rc = enqueue_cycle(pl, d_out, st))) return rc;
            ++done;
            CU(cudaStreamSynchronize(st));
        }
        if ((rc = enqueue_reports(pl, st))) return rc;
    }
    pl->pending = true;
    pl->pending_stream = st;
    return 0;
}

int b200p_solve_wait(b200p_plan *pl, b200p_report *h_reports) {
    if (!pl) return fail_arg(B200P_ERR_ARG, "null plan");
    if (!pl->pending) return fail_arg(B200P_ERR_STATE, "no solve is pending on this plan");
    pl->pending = false;
    CU(cudaStreamSynchronize(pl->pending_stream));
    if (!pl->pending_eager) {
        // kernels launched = front + report gather + one body pass per V-cycle that ran
        int cyc = 0;
        for (int p = 0; p < pl->P; ++p) cyc = std::max(cyc, pl->rep.cycles[p]);
        pl->launches += pl->g_solve.kernels + (int64_t)cyc * pl->cycle_kernels;
    }
    if (h_reports) read_reports(pl, h_reports);
    if (pl->profiling) prof_collect(pl);
    return 0;
}

int b200p_solve(b200p_plan *pl, const uint8_t *d_mask, const double *d_known, double *d_out,
                b200p_report *h_reports, void *stream) {
    int rc = b200p_solve_async(pl, d_mask, d_known, d_out, stream);
    if (rc) return rc;
    return b200p_solve_wait(pl, h_reports);
}

static int ensure_staging(b200p_plan *pl, bool u8) {
    const size_t plane = (size_t)pl->cfg.width * pl->cfg.height;
    if (!pl->d_in_mask) {
        int rc;
        if ((rc = dev_alloc(pl, &pl->d_in_mask, pl->F * plane))) return rc;
        if ((rc = dev_alloc(pl, &pl->d_in_known, pl->P * plane))) return rc;
        if ((rc = dev_alloc(pl, &pl->d_out, pl->P * plane))) return rc;
    }
    if (u8 && !pl->d_io_u8) {
        int rc;
        if ((rc = dev_alloc(pl, &pl->d_io_u8, pl->P * plane))) return rc;
    }
    if (!pl->own_stream) CU(cudaStreamCreateWithFlags(&pl->own_stream, cudaStreamNonBlocking));
    return 0;
}

static bool any_nonzero(const uint8_t *p, size_t n) {
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
        uint64_t v;
        memcpy(&v, p + i, 8);
        if (v) return true;
    }
    for (; i < n; ++i)
        if (p[i]) return true;
    return false;
}

static int check_masks(const b200p_plan *pl, const uint8_t *h_mask) {
    const size_t plane = (size_t)pl->cfg.width * pl->cfg.height;
    for (int f = 0; f < pl->F; ++f)
        if (!any_nonzero(h_mask + (size_t)f * plane, plane))
            return fail_arg(B200P_ERR_EMPTY_MASK, "cannot solve without known pixels");
    return 0;
}

// Known pixels of one frame: count, then indices (row-major order) -- the mask is ~98 % zeros at
// the benchmark densities, so whole 8-byte words are skipped.
static size_t count_nonzero(const uint8_t *m, size_t n) {
    size_t cnt = 0, i = 0;
    for (; i + 8 <= n; i += 8) {
        uint64_t v;
        memcpy(&v, m + i, 8);
        if (!v) continue;
        for (int k = 0; k < 8; ++k) cnt += m[i + k] != 0;
    }
    for (; i < n; ++i) cnt += m[i] != 0;
    return cnt;
}

static size_t list_nonzero(const uint8_t *m, size_t n, uint32_t *idx) {
    size_t cnt = 0, i = 0;
    for (; i + 8 <= n; i += 8) {
        uint64_t v;
        memcpy(&v, m + i, 8);
        if (!v) continue;
        for (int k = 0; k < 8; ++k)
            if (m[i + k]) idx[cnt++] = (uint32_t)(i + k);
    }
    for (; i < n; ++i)
        if (m[i]) idx[cnt++] = (uint32_t)i;
    return cnt;
}

// A small process-wide pool for the host-side gather of the sparse ingest (the only host loop of the library that
// touches whole planes).  B200P_HOST_THREADS workers (default min(8, cores)); the caller works too.  Never destroyed:
// its threads sleep on a condition variable between calls.
class HostPool {
    std::mutex m, callers;
    std::condition_variable cv, done_cv;
    const std::function<void(int)> *job = nullptr;
    int ntasks = 0, pending = 0, workers = 0;
    std::atomic<int> next{0};
    uint64_t gen = 0;
    void loop() {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> lk(m);
        for (;;) {
            cv.wait(lk, [&] { return gen != seen; });
            seen = gen;
            const std::function<void(int)> *f = job;
            const int n = ntasks;
            lk.unlock();
            for (int t; (t = next.fetch_add(1)) < n;) (*f)(t);
            lk.lock();
            if (--pending == 0) done_cv.notify_one();
        }
    }
public:
    explicit HostPool(int n) : workers(n) {
        for (int i = 0; i < n; ++i) std::thread([this] { loop(); }).detach();
    }
    int width() const { return workers + 1; }
    void run(int n, const std::function<void(int)> &f) {
        std::lock_guard<std::mutex> one(callers);
        {
            std::lock_guard<std::mutex> lk(m);
            job = &f;
            ntasks = n;
            next = 0;
            pending = workers;
            ++gen;
        }
        cv.notify_all();
        for (int t; (t = next.fetch_add(1)) < n;) f(t);
        std::unique_lock<std::mutex> lk(m);
        done_cv.wait(lk, [&] { return pending == 0; });
    }
};
static HostPool &host_pool() {
    static HostPool *pool = [] {
        const char *e = getenv("B200P_HOST_THREADS");
        int n = e ? atoi(e) : (int)std::min(8u, std::max(1u, std::thread::hardware_concurrency()));
        return new HostPool(std::max(0, n - 1));
    }();
    return *pool;
}

static int ensure_sparse_staging(b200p_plan *pl, size_t entries) {
    if (entries <= pl->sp_cap) return 0;
    const size_t cap = entries + entries / 4 + 1024;
    const int C = pl->cfg.channels;
    // (h_cnt / d_cnt belong to the pinned zero-copy ingest and are not touched here)
    if (pl->h_sp_idx) cudaFreeHost(pl->h_sp_idx);
    if (pl->h_sp_val) cudaFreeHost(pl->h_sp_val);
    if (pl->d_sp_idx) cudaFree(pl->d_sp_idx);
    if (pl->d_sp_val) cudaFree(pl->d_sp_val);
    pl->h_sp_idx = pl->d_sp_idx = nullptr;
    pl->h_sp_val = pl->d_sp_val = nullptr;
    pl->sp_cap = 0;
    CU(cudaMallocHost((void **)&pl->h_sp_idx, cap * sizeof(uint32_t)));
    CU(cudaMallocHost((void **)&pl->h_sp_val, cap * C * sizeof(double)));
    CU(cudaMalloc((void **)&pl->d_sp_idx, cap * sizeof(uint32_t)));
    CU(cudaMalloc((void **)&pl->d_sp_val, cap * C * sizeof(double)));
    pl->sp_cap = cap;
    return 0;
}

// Host f64 entry point.  The path uses `known` only at mask pixels (rhs = where(mask, known, 0),
// core.py:147-151), so when the mask is sparse the H2D side carries the mask plane plus the values
// at mask pixels only: 4K RGB at 2 % moves 12 MB instead of 207 MB per frame.
//   * `h_known` pinned (cudaHostAlloc / cudaHostRegister): a kernel reads those values straight
//     from the caller's array over PCIe (zero copy) and writes the zero-filled known plane;
//   * pageable `h_known`: this thread gathers a compacted (pixel index, C values) list into
//     pinned staging, and a scatter kernel rebuilds the plane.
// Dense masks (list larger than half the planes) and B200P_DENSE_INGEST=1 copy the planes as they
// are.  The result is copied back in full.
int b200p_solve_host_async(b200p_plan *pl, const uint8_t *h_mask, const double *h_known, double *h_out) {
    if (!pl || !h_mask || !h_known || !h_out) return fail_arg(B200P_ERR_ARG, "null argument");
    if (pl->pending) return fail_arg(B200P_ERR_STATE, "a solve is already pending on this plan");
    int rc = check_masks(pl, h_mask);
    if (rc) return rc;
    const size_t plane = (size_t)pl->cfg.width * pl->cfg.height;
    const int C = pl->cfg.channels;
    const char *env_dense = getenv("B200P_DENSE_INGEST");  // read per call (A/B tests toggle it)
    const bool force_dense = pl->ingest_mode == 1 || (env_dense && atoi(env_dense) != 0);
    if ((rc = ensure_staging(pl, false))) return rc;
    cudaStream_t st = pl->own_stream;
    const size_t dense_bytes = pl->P * plane * sizeof(double);
    CU(cudaMemcpyAsync(pl->d_in_mask, h_mask, pl->F * plane, cudaMemcpyHostToDevice, st));
    pl->last_h2d = (int64_t)(pl->F * plane + dense_bytes);
    pl->last_h2d_counted = false;
    // pinned source: the device fetches the mask pixels' values itself (no host pass over `known`)
    const double *mapped = nullptr;
    if (!force_dense && pl->ingest_mode != 2) {
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, h_known) == cudaSuccess && at.type == cudaMemoryTypeHost &&
            at.devicePointer)
            mapped = static_cast<const double *>(at.devicePointer);
        else
            cudaGetLastError();
    }
    bool done = false;
    if (mapped) {
        // density from a strided sample of the mask words (the choice of path does not change results)
        size_t seen = 0, hit = 0;
        const size_t n = pl->F * plane;
        for (size_t i = 0; i + 8 <= n; i += 8 * 61) {
            for (int k = 0; k < 8; ++k) hit += h_mask[i + k] != 0;
            seen += 8;
        }
        if (seen && hit * 4 <= seen) {  // <= 25 % known pixels: fetching them beats copying the planes
            if (!pl->h_cnt) {
                CU(cudaHostAlloc((void **)&pl->h_cnt, 64, cudaHostAllocMapped));
                CU(cudaMalloc((void **)&pl->d_cnt, 64));
            }
            CU(cudaMemsetAsync(pl->d_cnt, 0, 8, st));
            {
                LaunchScope sc(pl, st, KK_CONVERT, (double)(n + dense_bytes));
                gather_known_mapped_kernel<<<(unsigned)((n + ST_THREADS - 1) / ST_THREADS), ST_THREADS, 0, st>>>(
                    pl->d_in_mask, mapped, n, C, plane, pl->d_in_known, pl->d_cnt);
                CU(cudaGetLastError());
            }
            {
                LaunchScope sc(pl, st, KK_CONVERT, 16.0);
                publish_count_kernel<<<1, 1, 0, st>>>(pl->d_cnt, pl->h_cnt);
                CU(cudaGetLastError());
            }
            pl->last_h2d_counted = true;  // F*plane + count*C*8, known once the stream has run
            done = true;
        }
    }
    if (!done && !force_dense && plane < (1ull << 32)) {
        // pageable source (or B200P ingest mode 2): the host gathers a (pixel index, C values) list into pinned
        // staging -- every frame cut into row chunks that the host pool counts, then lists and gathers in place
        const int h = pl->cfg.height, w = pl->cfg.width;
        const int chunks = std::max(1, std::min(h, 4 * host_pool().width() / std::max(1, std::min(pl->F, 4))));
        const int ntask = pl->F * chunks;
        std::vector<size_t> cnt(ntask + 1, 0);
        auto rows_of = [&](int t, size_t &lo, size_t &n) {
            const int c = t % chunks;
            const size_t r0 = (size_t)h * c / chunks, r1 = (size_t)h * (c + 1) / chunks;
            lo = r0 * w;
            n = (r1 - r0) * w;
        };
        const std::function<void(int)> count = [&](int t) {
            size_t lo, n;
            rows_of(t, lo, n);
            cnt[t + 1] = count_nonzero(h_mask + (size_t)(t / chunks) * plane + lo, n);
        };
        host_pool().run(ntask, count);
        for (int t = 0; t < ntask; ++t) cnt[t + 1] += cnt[t];   // offsets
        const size_t total = cnt[ntask];
        const size_t sparse_bytes = total * (sizeof(uint32_t) + C * sizeof(double));
        if (sparse_bytes * 2 <= dense_bytes) {
            if ((rc = ensure_sparse_staging(pl, total))) return rc;
            CU(cudaMemsetAsync(pl->d_in_known, 0, dense_bytes, st));
            const std::function<void(int)> gather = [&](int t) {
                size_t lo, n;
                rows_of(t, lo, n);
                const int f = t / chunks;
                uint32_t *idx = pl->h_sp_idx + cnt[t];
                double *val = pl->h_sp_val + cnt[t] * C;
                const size_t k_n = list_nonzero(h_mask + (size_t)f * plane + lo, n, idx);
                for (size_t k = 0; k < k_n; ++k) idx[k] += (uint32_t)lo;
                for (int c = 0; c < C; ++c) {
                    const double *src = h_known + ((size_t)f * C + c) * plane;
                    for (size_t k = 0; k < k_n; ++k) val[k * C + c] = src[idx[k]];
                }
            };
            host_pool().run(ntask, gather);
            CU(cudaMemcpyAsync(pl->d_sp_idx, pl->h_sp_idx, total * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
            CU(cudaMemcpyAsync(pl->d_sp_val, pl->h_sp_val, total * C * sizeof(double), cudaMemcpyHostToDevice, st));
            for (int f = 0; f < pl->F; ++f) {
                const size_t off = cnt[f * chunks], n = (cnt[(f + 1) * chunks] - off) * C;
                if (!n) continue;
                LaunchScope sc(pl, st, KK_CONVERT, 20.0 * n);
                scatter_known_kernel<<<(unsigned)((n + ST_THREADS - 1) / ST_THREADS), ST_THREADS, 0, st>>>(
                    pl->d_sp_idx + off, pl->d_sp_val + off * C, n, C, plane, pl->d_in_known + (size_t)f * C * plane);
                CU(cudaGetLastError());
            }
            pl->last_h2d = (int64_t)(pl->F * plane + sparse_bytes);
            done = true;
        }
    }
    if (!done) CU(cudaMemcpyAsync(pl->d_in_known, h_known, dense_bytes, cudaMemcpyHostToDevice, st));
    if ((rc = b200p_solve_async(pl, pl->d_in_mask, pl->d_in_known, pl->d_out, st))) return rc;
    CU(cudaMemcpyAsync(h_out, pl->d_out, dense_bytes, cudaMemcpyDeviceToHost, st));
    pl->last_d2h = (int64_t)dense_bytes;
    return 0;
}

int b200p_plan_set_ingest(b200p_plan *pl, int mode) {
    if (!pl) return fail_arg(B200P_ERR_ARG, "null plan");
    if (mode < 0 || mode > 2)
        return fail_arg(B200P_ERR_ARG, "ingest mode must be 0 (auto), 1 (dense) or 2 (host gather), got %d", mode);
    pl->ingest_mode = mode;
    return 0;
}

int b200p_plan_last_transfer_bytes(const b200p_plan *pl, int64_t *h2d, int64_t *d2h) {
    if (!pl) return fail_arg(B200P_ERR_ARG, "null plan");
    if (pl->pending) return fail_arg(B200P_ERR_STATE, "a solve is pending on this plan: call b200p_solve_wait first");
    if (h2d)
        *h2d = pl->last_h2d_counted
                   ? (int64_t)((size_t)pl->F * pl->cfg.width * pl->cfg.height +
                               *pl->h_cnt * (size_t)pl->cfg.channels * sizeof(double))
                   : pl->last_h2d;
    if (d2h) *d2h = pl->last_d2h;
    return 0;
}

int b200p_solve_host(b200p_plan *pl, const uint8_t *h_mask, const double *h_known, double *h_out,
                     b200p_report *h_reports) {
    int rc = b200p_solve_host_async(pl, h_mask, h_known, h_out);
    if (rc) return rc;
    return b200p_solve_wait(pl, h_reports);
}

int b200p_solve_host_u8_async(b200p_plan *pl, const uint8_t *h_mask, const uint8_t *h_known_u8,
                              uint8_t *h_out_u8) {
    if (!pl || !h_mask || !h_known_u8 || !h_out_u8) return fail_arg(B200P_ERR_ARG, "null argument");
    int rc = check_masks(pl, h_mask);
    if (rc) return rc;
    if ((rc = ensure_staging(pl, true))) return rc;
    const size_t plane = (size_t)pl->cfg.width * pl->cfg.height;
    const size_t n = pl->P * plane;
    cudaStream_t st = pl->own_stream;
    CU(cudaMemcpyAsync(pl->d_in_mask, h_mask, pl->F * plane, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(pl->d_io_u8, h_known_u8, n, cudaMemcpyHostToDevice, st));
    {
        LaunchScope sc(pl, st, KK_CONVERT, 9.0 * n);
        u8_to_f64_kernel<<<(unsigned)((n + ST_THREADS - 1) / ST_THREADS), ST_THREADS, 0, st>>>(
            pl->d_io_u8, n, pl->d_in_known);
        CU(cudaGetLastError());
    }
    if ((rc = b200p_solve_async(pl, pl->d_in_mask, pl->d_in_known, pl->d_out, st))) return rc;
    {
        LaunchScope sc(pl, st, KK_CONVERT, 9.0 * n);
        f64_to_u8_kernel<<<(unsigned)((n + ST_THREADS - 1) / ST_THREADS), ST_THREADS, 0, st>>>(
            pl->d_out, n, pl->d_io_u8);
        CU(cudaGetLastError());
    }
    CU(cudaMemcpyAsync(h_out_u8, pl->d_io_u8, n, cudaMemcpyDeviceToHost, st));
    pl->last_h2d = (int64_t)(pl->F * plane + n);
    pl->last_d2h = (int64_t)n;
    return 0;
}

int b200p_solve_host_u8(b200p_plan *pl, const uint8_t *h_mask, const uint8_t *h_known_u8,
                        uint8_t *h_out_u8, b200p_report *h_reports) {
    int rc = b200p_solve_host_u8_async(pl, h_mask, h_known_u8, h_out_u8);
    if (rc) return rc;
    return b200p_solve_wait(pl, h_reports);
}

// 8-bit image files as they are on disk: interleaved pixels (F, h, w, C) as ImageFile holds
// them (fileio.py:27-55) and the bit-packed P4 raster of write_mask / read_mask (fileio.py:181-230: rows
// padded to bytes, MSB first, 1 = known).  Unpacking, channel_fields and image_from_fields run on the
// device; the round / clip / interleave of the result rides on the last combine pass of the solve.
static int check_mask_bits(const b200p_plan *pl, const uint8_t *bits) {
    const int w = pl->cfg.width, h = pl->cfg.height, rb = (w + 7) / 8;
    const uint8_t last = (w % 8) ? (uint8_t)(0xff00u >> (w % 8)) : 0xff;   // padding bits of a row are ignored
    for (int f = 0; f < pl->F; ++f) {
        bool any = false;
        const uint8_t *fp = bits + (size_t)f * h * rb;
        for (int y = 0; y < h && !any; ++y) {
            const uint8_t *row = fp + (size_t)y * rb;
            any = (rb > 1 && any_nonzero(row, rb - 1)) || (row[rb - 1] & last);
        }
        if (!any) return fail_arg(B200P_ERR_EMPTY_MASK, "cannot solve without known pixels");
    }
    return 0;
}

int b200p_solve_host_image_u8_async(b200p_plan *pl, const uint8_t *h_mask_bits, const uint8_t *h_pixels,
                                    uint8_t *h_out) {
    if (!pl || !h_mask_bits || !h_pixels || !h_out) return fail_arg(B200P_ERR_ARG, "null argument");
    if (pl->pending) return fail_arg(B200P_ERR_STATE, "a solve is already pending on this plan");
    int rc = check_mask_bits(pl, h_mask_bits);
    if (rc) return rc;
    if ((rc = ensure_staging(pl, true))) return rc;
    const int w = pl->cfg.width, h = pl->cfg.height, rb = (w + 7) / 8;
    const size_t plane = (size_t)w * h, npix = pl->F * plane, n = pl->P * plane;
    const size_t nbits = (size_t)pl->F * h * rb;
    if (!pl->d_mask_bits && (rc = dev_alloc(pl, &pl->d_mask_bits, nbits))) return rc;
    cudaStream_t st = pl->own_stream;
    CU(cudaMemcpyAsync(pl->d_mask_bits, h_mask_bits, nbits, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(pl->d_io_u8, h_pixels, n, cudaMemcpyHostToDevice, st));
    {
        LaunchScope sc(pl, st, KK_CONVERT, (double)(nbits + npix));
        unpack_mask_bits_kernel<<<(unsigned)((nbits + ST_THREADS - 1) / ST_THREADS), ST_THREADS, 0, st>>>(
            pl->d_mask_bits, nbits, w, rb, pl->d_in_mask);
        CU(cudaGetLastError());
    }
    {
        LaunchScope sc(pl, st, KK_CONVERT, 9.0 * n);
        deinterleave_u8_kernel<<<(unsigned)((npix + ST_THREADS - 1) / ST_THREADS), ST_THREADS, 0, st>>>(
            pl->d_io_u8, npix, pl->C, plane, pl->d_in_known);
        CU(cudaGetLastError());
    }
    // the pixels have been consumed: the same buffer receives the decoded image
    if ((rc = solve_async_impl(pl, pl->d_in_mask, pl->d_in_known, pl->d_out, pl->d_io_u8, st))) return rc;
    CU(cudaMemcpyAsync(h_out, pl->d_io_u8, n, cudaMemcpyDeviceToHost, st));
    pl->last_h2d = (int64_t)(nbits + n);
    pl->last_h2d_counted = false;
    pl->last_d2h = (int64_t)n;
    return 0;
}

int b200p_solve_host_image_u8(b200p_plan *pl, const uint8_t *h_mask_bits, const uint8_t *h_pixels,
                              uint8_t *h_out, b200p_report *h_reports) {
    int rc = b200p_solve_host_image_u8_async(pl, h_mask_bits, h_pixels, h_out);
    if (rc) return rc;
    return b200p_solve_wait(pl, h_reports);
}

// ---- stage entry points -------------------------------------------------

int b200p_plan_build_hierarchy(b200p_plan *pl, const uint8_t *d_mask, const double *d_known,
                               void *stream) {
    if (!pl || !d_mask || !d_known) return fail_arg(B200P_ERR_ARG, "null argument");
    bind_level0(pl, d_mask, d_known);
    int rc = enqueue_hierarchy(pl, (cudaStream_t)stream);
    if (rc) return rc;
    pl->hierarchy_ready = true;
    return 0;
}

int b200p_plan_level_ptrs(const b200p_plan *pl, int level, const uint8_t **d_mask,
                          const double **d_rhs) {
    if (!pl || level < 0 || level >= (int)pl->lev.size()) return fail_arg(B200P_ERR_ARG, "bad level %d", level);
    if (!pl->hierarchy_ready) return fail_arg(B200P_ERR_STATE, "build_hierarchy has not run");
    if (d_mask) *d_mask = pl->lev[level].d_mask;
    if (d_rhs) *d_rhs = level == 0 ? nullptr : pl->lev[level].d_rhs;
    return 0;
}

int b200p_plan_history(b200p_plan *pl, int problem, double *h_out, int cap) {
    if (!pl || !h_out) return fail_arg(B200P_ERR_ARG, "null argument");
    if (problem < 0 || problem >= pl->P) return fail_arg(B200P_ERR_ARG, "bad problem index %d", problem);
    if (cap < 0) return fail_arg(B200P_ERR_ARG, "bad capacity %d", cap);
    const int n = std::min(cap, pl->hist_cap);
    CU(cudaMemcpy(h_out, pl->d_hist + (size_t)problem * pl->hist_cap, sizeof(double) * (size_t)n,
                  cudaMemcpyDeviceToHost));
    return n;
}

int b200p_plan_set_step_callback(b200p_plan *pl, b200p_step_fn fn, void *user) {
    if (!pl) return fail_arg(B200P_ERR_ARG, "null argument");
    pl->step_cb = fn;
    pl->step_user = fn ? user : nullptr;
    return 0;
}

int b200p_plan_cascade(b200p_plan *pl, double *d_u, void *stream) {
    if (!pl || !d_u) return fail_arg(B200P_ERR_ARG, "null argument");
    if (!pl->hierarchy_ready) return fail_arg(B200P_ERR_STATE, "build_hierarchy has not run");
    cudaStream_t st = (cudaStream_t)stream;
    int rc = launch_set_int(pl, pl->d_units, pl->P, 0, st);
    if (rc) return rc;
    if (pl->cfg.smoother == 1) return cg_cascade_stage(pl, d_u, st);
    return enqueue_cascade(pl, d_u, st);
}

int b200p_plan_vcycle(b200p_plan *pl, int level, double *d_u, const double *d_rhs, int *h_fine_units,
                      void *stream) {
    if (!pl || !d_u || !d_rhs) return fail_arg(B200P_ERR_ARG, "null argument");
    if (level < 0 || level >= (int)pl->lev.size()) return fail_arg(B200P_ERR_ARG, "bad level %d", level);
    if (!pl->hierarchy_ready) return fail_arg(B200P_ERR_STATE, "build_hierarchy has not run");
    cudaStream_t st = (cudaStream_t)stream;
    int rc = launch_set_int(pl, pl->d_units, pl->P, 0, st);
    if (rc) return rc;
    if (pl->cfg.smoother == 1) {
        // CG-smoothed cycle (multigrid.py:278-279, 335-371): in place on d_u, units counted at level 0
        if ((rc = cg_vcycle(pl, level, d_u, d_rhs, false, nullptr, pl->d_units, st))) return rc;
    } else {
        UBuf u;
        u.cur = d_u;
        u.alt = pl->lev[level].d_u_alt;
        if ((rc = enqueue_vcycle(pl, level, u, d_rhs, false, nullptr, pl->d_units, false, st))) return rc;
    }
    if (h_fine_units) {
        CU(cudaMemcpyAsync(h_fine_units, pl->d_units, pl->P * sizeof(int), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (level != 0) memset(h_fine_units, 0, pl->P * sizeof(int));
    }
    return 0;
}

int b200p_plan_oras_sweeps(b200p_plan *pl, int level, const double *d_b, double *d_u, int max_sweeps,
                           double stop_norm, int path, int *h_sweeps, double *h_rn, void *stream) {
    if (!pl || !d_b || !d_u) return fail_arg(B200P_ERR_ARG, "null argument");
    if (level < 0 || level >= (int)pl->lev.size()) return fail_arg(B200P_ERR_ARG, "bad level %d", level);
    if (!pl->lev[level].d_mask) return fail_arg(B200P_ERR_STATE, "level mask not bound (build_hierarchy)");
    LevelHost &L = pl->lev[level];
    int force = -1;  // plan default
    const bool is32 = L.info.block_w == 32 && L.info.block_h == 32;
    const bool is16 = L.info.block_w == 16 && L.info.block_h == 16;
    const bool is8 = L.info.block_w == 8 && L.info.block_h == 8;
    if (path == 1) force = TILE_GENERIC;
    else if (path == 2) {
        force = tile_for(L.info.block_w, L.info.block_h);
        if (force == TILE_GENERIC)
            return fail_arg(B200P_ERR_UNSUPPORTED, "level %d has no register-tile kernel", level);
    } else if (path == 3) {
        if (!L.fused) return fail_arg(B200P_ERR_UNSUPPORTED, "level %d is not eligible for the fused sweep", level);
        force = -2;
    } else if (path >= 10) {
        const int t = path - 10;
        const bool lab32 = t == TILE_32_A || t == TILE_32_C || t == TILE_32_S || t == TILE_32_T || t == TILE_32_U ||
                           t == TILE_32_TMA || t == TILE_32_L || t == TILE_32_WQ;
        if (is32 && lab32 && !B200P_LAB)
            return fail_arg(B200P_ERR_UNSUPPORTED, "tile variant %d is an experiment: build with -DB200P_EXPERIMENTS", t);
        const bool ok = (is32 && (lab32 || t == TILE_32_B || t == TILE_32_W)) || (is16 && t == TILE_16) ||
                        (is8 && t == TILE_8);
        if (!ok) return fail_arg(B200P_ERR_UNSUPPORTED, "level %d is not eligible for tile variant %d", level, t);
        force = t;
    } else if (path != 0) {
        return fail_arg(B200P_ERR_ARG, "unknown path %d", path);
    }
    UBuf ub;
    ub.cur = d_u;
    ub.alt = L.d_u_alt;
    cudaStream_t st = (cudaStream_t)stream;
    int rc;
    if ((rc = launch_set_int(pl, pl->d_gate, pl->P, 1, st))) return rc;
    if ((rc = launch_set_int(pl, pl->d_sweeps, pl->P, 0, st))) return rc;
    if (path == 0 && stop_norm == 0.0 && L.nblocks == 1 && level == (int)pl->lev.size() - 1) {
        // a single-block coarsest level is what the solve drivers hand to K7 (sweeps looped in one kernel,
        // multigrid.py:264-279 with stop_norm = 0): the default path of the stage call runs the same kernel,
        // so that a single-level V-cycle and its sweeps are the same arithmetic (tests/test_multigrid.py:218-233)
        if ((rc = launch_coarse(pl, L, d_u, d_b, false, 2, 0.0, max_sweeps, nullptr, pl->d_sweeps, 0, st))) return rc;
        if ((rc = launch_norm(pl, L, d_u, d_b, false, false, nullptr, st))) return rc;
        {
            LaunchScope sc(pl, st, KK_CONTROL, 0.0);
            sweep_gate_kernel<<<(pl->P + 127) / 128, 128, 0, st>>>(pl->P, pl->d_rs, 0.0, 0, pl->d_gate,
                                                                   pl->d_sweeps, pl->d_rn, pl->d_any);
            CU(cudaGetLastError());
        }
        if (h_sweeps) CU(cudaMemcpyAsync(h_sweeps, pl->d_sweeps, pl->P * sizeof(int), cudaMemcpyDeviceToHost, st));
        if (h_rn) CU(cudaMemcpyAsync(h_rn, pl->d_rn, pl->P * sizeof(double), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (pl->profiling) prof_collect(pl);
        return 0;
    }
    int it = 0;
    for (;;) {
        const int chunk = 8;
        if ((rc = launch_set_int(pl, pl->d_any, 1, 0, st))) return rc;
        for (int k = 0; k < chunk && it <= max_sweeps; ++k, ++it) {
            if ((rc = launch_norm(pl, L, ub.cur, d_b, false, false, pl->d_gate, st))) return rc;
            {
                LaunchScope sc(pl, st, KK_CONTROL, 0.0);
                sweep_gate_kernel<<<(pl->P + 127) / 128, 128, 0, st>>>(
                    pl->P, pl->d_rs, stop_norm, max_sweeps, pl->d_gate, pl->d_sweeps, pl->d_rn, pl->d_any);
                CU(cudaGetLastError());
            }
            if ((rc = launch_sweep(pl, L, ub, d_b, false, pl->d_gate, pl->d_sweeps, force, st))) return rc;
        }
        CU(cudaMemcpyAsync(pl->h_any, pl->d_any, sizeof(int), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (!*pl->h_any || it > max_sweeps) break;
    }
    if ((rc = settle(pl, L, ub, d_u, st))) return rc;
    if (h_sweeps) CU(cudaMemcpyAsync(h_sweeps, pl->d_sweeps, pl->P * sizeof(int), cudaMemcpyDeviceToHost, st));
    if (h_rn) CU(cudaMemcpyAsync(h_rn, pl->d_rn, pl->P * sizeof(double), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (pl->profiling) prof_collect(pl);
    return 0;
}

int b200p_plan_solve_blocks(b200p_plan *pl, int level, const double *d_r, double target_sq,
                            double *d_v, void *stream) {
    if (!pl || !d_r || !d_v) return fail_arg(B200P_ERR_ARG, "null argument");
    if (level < 0 || level >= (int)pl->lev.size()) return fail_arg(B200P_ERR_ARG, "bad level %d", level);
    if (!pl->lev[level].d_mask) return fail_arg(B200P_ERR_STATE, "level mask not bound (build_hierarchy)");
    LevelHost &L = pl->lev[level];
    SweepArgs A;
    A.L = L.dev;
    A.u = d_r;
    A.b = nullptr;
    A.mask = L.d_mask;
    A.channels = pl->C;
    A.plane = (size_t)L.info.height * L.info.width;
    A.pred = nullptr;
    A.rs = nullptr;
    A.mflag = nullptr;
    A.eta = target_sq;
    A.max_iters = local_cap(pl, L);
    A.scratch = d_v;
    cudaStream_t st = (cudaStream_t)stream;
    LaunchScope sc(pl, st, KK_SWEEP, 0.0);
    oras_sweep_generic_kernel<false, 1><<<dim3(L.nblocks, pl->P), GEN_THREADS,
                                          smem_cg_bytes(L.info.block_w, L.info.block_h), st>>>(A);
    CU(cudaGetLastError());
    return 0;
}

int b200p_plan_scatter_weighted(b200p_plan *pl, int level, const double *d_v, double *d_field, void *stream) {
    if (!pl || !d_v || !d_field) return fail_arg(B200P_ERR_ARG, "null argument");
    if (level < 0 || level >= (int)pl->lev.size()) return fail_arg(B200P_ERR_ARG, "bad level %d", level);
    LevelHost &L = pl->lev[level];
    cudaStream_t st = (cudaStream_t)stream;
    const size_t plane = (size_t)L.info.height * L.info.width;
    const size_t n = (size_t)pl->P * L.nblocks * L.info.block_w * L.info.block_h;
    // the plan's tile scratch receives (v * wy) * wx, then the combine pass of the sweeps (K2b) sums the
    // covering tiles of every pixel in ascending block order onto a zero field (np.bincount order)
    weight_tiles_kernel<<<(unsigned)((n + ST_THREADS_COMBINE - 1) / ST_THREADS_COMBINE), ST_THREADS_COMBINE, 0, st>>>(
        L.dev, d_v, pl->d_scratch, n);
    CU(cudaGetLastError());
    fill_double_kernel<<<(pl->P + 127) / 128, 128, 0, st>>>(pl->d_rs, pl->P, 1.0);   // every problem is live
    CU(cudaGetLastError());
    CU(cudaMemsetAsync(d_field, 0, sizeof(double) * pl->P * plane, st));
    dim3 g((L.info.width + ST_THREADS_COMBINE - 1) / ST_THREADS_COMBINE,
           (L.info.height + COMBINE_ROWS - 1) / COMBINE_ROWS, pl->P);
    LaunchScope sc(pl, st, KK_COMBINE, field_bytes(pl, L, 3.0, 0.0));
    oras_combine_kernel<<<g, ST_THREADS_COMBINE, 0, st>>>(L.dev, pl->d_scratch, plane, nullptr, pl->d_rs, d_field,
                                                          nullptr, 0, L.info.height, nullptr, pl->C);
    CU(cudaGetLastError());
    return 0;
}

int b200p_apply(const uint8_t *d_mask, int h, int w, double spacing, const double *d_u, double *d_out,
                void *stream) {
    if (!d_mask || !d_u || !d_out || h < 1 || w < 1) return fail_arg(B200P_ERR_ARG, "bad argument");
    if (!(spacing > 0.0)) return fail_arg(B200P_ERR_ARG, "spacing must be positive, got %g", spacing);
    const size_t n = (size_t)h * w;
    residual_field_kernel<<<(unsigned)((n + ST_THREADS - 1) / ST_THREADS), ST_THREADS, 0,
                            (cudaStream_t)stream>>>(d_u, nullptr, d_mask, h, w, 1.0 / (spacing * spacing),
                                                    1, d_out);
    CU(cudaGetLastError());
    return 0;
}

int b200p_residual(const uint8_t *d_mask, int h, int w, double spacing, const double *d_b,
                   const double *d_u, double *d_r, void *stream) {
    if (!d_mask || !d_u || !d_b || !d_r || h < 1 || w < 1) return fail_arg(B200P_ERR_ARG, "bad argument");
    if (!(spacing > 0.0)) return fail_arg(B200P_ERR_ARG, "spacing must be positive, got %g", spacing);
    const size_t n = (size_t)h * w;
    residual_field_kernel<<<(unsigned)((n + ST_THREADS - 1) / ST_THREADS), ST_THREADS, 0,
                            (cudaStream_t)stream>>>(d_u, d_b, d_mask, h, w, 1.0 / (spacing * spacing), 0,
                                                    d_r);
    CU(cudaGetLastError());
    return 0;
}

int b200p_residual_sqnorm(const uint8_t *d_mask, int h, int w, double spacing, const double *d_b,
                          const double *d_u, int planes, double *h_out, void *stream) {
    if (!d_mask || !d_u || !d_b || !h_out || h < 1 || w < 1 || planes < 1)
        return fail_arg(B200P_ERR_ARG, "bad argument");
    if (!(spacing > 0.0)) return fail_arg(B200P_ERR_ARG, "spacing must be positive, got %g", spacing);
    cudaStream_t st = (cudaStream_t)stream;
    const int ctas = 256;
    double *d_partial = nullptr, *d_rs = nullptr;
    int *d_pf = nullptr, *d_flag = nullptr;
    unsigned *d_cnt = nullptr;
    CU(cudaMalloc(&d_partial, sizeof(double) * ctas * planes));
    CU(cudaMalloc(&d_pf, sizeof(int) * ctas * planes));
    CU(cudaMalloc(&d_cnt, sizeof(unsigned) * planes));
    CU(cudaMalloc(&d_rs, sizeof(double) * planes));
    CU(cudaMalloc(&d_flag, sizeof(int) * planes));
    CU(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned) * planes, st));
    residual_sqnorm_kernel<false, false><<<dim3(ctas, planes), ST_THREADS, 0, st>>>(
        d_u, d_b, d_mask, h, w, 1.0 / (spacing * spacing), planes, (size_t)h * w, nullptr, d_partial,
        d_pf, d_cnt, d_rs, d_flag);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_out, d_rs, sizeof(double) * planes, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d_partial); cudaFree(d_pf); cudaFree(d_cnt); cudaFree(d_rs); cudaFree(d_flag);
    if (e != cudaSuccess) return fail_cuda(e, "residual_sqnorm");
    return 0;
}

int b200p_image_from_fields(const double *d_fields, int frames, int channels, int h, int w, uint8_t *d_pixels,
                            void *stream) {
    if (!d_fields || !d_pixels || frames < 1 || channels < 1 || h < 1 || w < 1)
        return fail_arg(B200P_ERR_ARG, "bad argument");
    const size_t plane = (size_t)h * w, npix = (size_t)frames * plane;
    egress_u8_kernel<<<(unsigned)((npix + ST_THREADS - 1) / ST_THREADS), ST_THREADS, 0, (cudaStream_t)stream>>>(
        d_fields, npix, channels, plane, nullptr, 1, d_pixels);
    CU(cudaGetLastError());
    return 0;
}

int b200p_unpack_mask_bits(const uint8_t *d_bits, int frames, int h, int w, uint8_t *d_mask, void *stream) {
    if (!d_bits || !d_mask || frames < 1 || h < 1 || w < 1) return fail_arg(B200P_ERR_ARG, "bad argument");
    const int rb = (w + 7) / 8;
    const size_t nbits = (size_t)frames * h * rb;
    unpack_mask_bits_kernel<<<(unsigned)((nbits + ST_THREADS - 1) / ST_THREADS), ST_THREADS, 0, (cudaStream_t)stream>>>(
        d_bits, nbits, w, rb, d_mask);
    CU(cudaGetLastError());
    return 0;
}

int b200p_downsample_mask(const uint8_t *d_fine, int h, int w, uint8_t *d_coarse, void *stream) {
    if (!d_fine || !d_coarse || h < 1 || w < 1) return fail_arg(B200P_ERR_ARG, "bad argument");
    if (words8_ok(w, d_fine, d_coarse))
        downsample_mask8_kernel<<<grid2x(w / 16, (h + 1) / 2, 1), ST_THREADS, 0, (cudaStream_t)stream>>>(d_fine, h, w, d_coarse);
    else
        downsample_mask_kernel<<<grid2x((w + 1) / 2, (h + 1) / 2, 1), ST_THREADS, 0, (cudaStream_t)stream>>>(d_fine, h, w, d_coarse);
    CU(cudaGetLastError());
    return 0;
}

int b200p_downsample_values(const uint8_t *d_fine_mask, const uint8_t *d_coarse_mask,
                            const double *d_fine_rhs, int h, int w, int modified, double *d_coarse_rhs,
                            void *stream) {
    if (!d_fine_mask || !d_coarse_mask || !d_fine_rhs || !d_coarse_rhs || h < 1 || w < 1)
        return fail_arg(B200P_ERR_ARG, "bad argument");
    downsample_values_kernel<<<grid2x((w + 1) / 2, (h + 1) / 2, 1), ST_THREADS, 0, (cudaStream_t)stream>>>(
        d_fine_mask, d_coarse_mask, d_fine_rhs, h, w, 1, modified, d_coarse_rhs);
    CU(cudaGetLastError());
    return 0;
}

int b200p_residual_restrict(const uint8_t *d_fine_mask, const uint8_t *d_coarse_mask, int h, int w,
                            double spacing, const double *d_b, const double *d_u, double *d_coarse_r,
                            void *stream) {
    if (!d_fine_mask || !d_coarse_mask || !d_b || !d_u || !d_coarse_r || h < 1 || w < 1)
        return fail_arg(B200P_ERR_ARG, "bad argument");
    if (!(spacing > 0.0)) return fail_arg(B200P_ERR_ARG, "spacing must be positive, got %g", spacing);
    residual_restrict_kernel<false><<<grid2x((w + 1) / 2, (h + 1) / 2, 1), ST_THREADS, 0,
                                      (cudaStream_t)stream>>>(
        d_u, d_b, d_fine_mask, d_coarse_mask, h, w, 1.0 / (spacing * spacing), 1, nullptr, d_coarse_r,
        nullptr);
    CU(cudaGetLastError());
    return 0;
}

int b200p_restrict_residual(const double *d_fine_r, const uint8_t *d_coarse_mask, int h, int w,
                            double *d_coarse_r, void *stream) {
    if (!d_fine_r || !d_coarse_mask || !d_coarse_r || h < 1 || w < 1)
        return fail_arg(B200P_ERR_ARG, "bad argument");
    restrict_field_kernel<<<grid2x((w + 1) / 2, (h + 1) / 2, 1), ST_THREADS, 0, (cudaStream_t)stream>>>(
        d_fine_r, d_coarse_mask, h, w, d_coarse_r);
    CU(cudaGetLastError());
    return 0;
}

int b200p_prolongate_correct(const double *d_coarse_e, const uint8_t *d_fine_mask, int h, int w,
                             double *d_u, void *stream) {
    if (!d_coarse_e || !d_fine_mask || !d_u || h < 1 || w < 1) return fail_arg(B200P_ERR_ARG, "bad argument");
    return launch_prolongate<false>(d_coarse_e, d_fine_mask, nullptr, h, w, 1, 1, nullptr, d_u, 0, 1 << 30, (cudaStream_t)stream);
}

int b200p_prolongate_solution(const double *d_coarse_u, const uint8_t *d_fine_mask,
                              const double *d_fine_rhs, int h, int w, double *d_u, void *stream) {
    if (!d_coarse_u || !d_fine_mask || !d_fine_rhs || !d_u || h < 1 || w < 1)
        return fail_arg(B200P_ERR_ARG, "bad argument");
    return launch_prolongate<true>(d_coarse_u, d_fine_mask, d_fine_rhs, h, w, 1, 1, nullptr, d_u, 0, 1 << 30, (cudaStream_t)stream);
}

// ---- device-memory helpers -----------------------------------------------
int b200p_malloc(void **d_ptr, int64_t bytes) {
    if (!d_ptr || bytes < 0) return fail_arg(B200P_ERR_ARG, "bad argument");
    CU(cudaMalloc(d_ptr, (size_t)std::max<int64_t>(bytes, 1)));
    return 0;
}
int b200p_free(void *d_ptr) {
    CU(cudaFree(d_ptr));
    return 0;
}

// ---- CUDA IPC: another process (one process per GPU, or several on one GPU) maps this buffer and
// reads / writes it through NVLink / peer memory.  d_ptr must be the base of a cudaMalloc allocation
// (b200p_malloc, or the plan-owned fields).
int b200p_ipc_export(const void *d_ptr, unsigned char handle[64]) {
    if (!d_ptr || !handle) return fail_arg(B200P_ERR_ARG, "null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, const_cast<void *>(d_ptr)));
    memcpy(handle, &h, 64);
    return 0;
}
int b200p_ipc_open(const unsigned char handle[64], void **d_ptr) {
    if (!d_ptr || !handle) return fail_arg(B200P_ERR_ARG, "null argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    CU(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return 0;
}
int b200p_ipc_close(void *d_ptr) {
    CU(cudaIpcCloseMemHandle(d_ptr));
    return 0;
}
int b200p_memcpy_d2d_async(void *d_dst, const void *d_src, int64_t bytes, void *stream) {
    CU(cudaMemcpyAsync(d_dst, d_src, (size_t)bytes, cudaMemcpyDefault, (cudaStream_t)stream));
    return 0;
}
int b200p_memcpy_h2d(void *d_dst, const void *h_src, int64_t bytes) {
    CU(cudaMemcpy(d_dst, h_src, (size_t)bytes, cudaMemcpyHostToDevice));
    return 0;
}
int b200p_memcpy_d2h(void *h_dst, const void *d_src, int64_t bytes) {
    CU(cudaMemcpy(h_dst, d_src, (size_t)bytes, cudaMemcpyDeviceToHost));
    return 0;
}
int b200p_memset(void *d_ptr, int value, int64_t bytes) {
    CU(cudaMemset(d_ptr, value, (size_t)bytes));
    return 0;
}
int b200p_device_synchronize(void) {
    CU(cudaDeviceSynchronize());
    return 0;
}

}  // extern "C"
