// qvg_engine.cu — libqvg.so: the C-ABI (include/qvg.h) over the sm_100a
// kernels in qvg_kernels.cuh and the pass planner in qvg_plan.hpp.
//
// Replaces, for the GPU strategy, the reference's block store + window +
// paired kernel + thread pool (reference store.cpp, cache.cpp, kernel.cpp,
// parallel.cpp): the state stays resident in HBM for the whole circuit and
// each planned pass is one kernel launch on the state's stream.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <functional>
#include <type_traits>
#include <memory>
#include <vector>

#include "qvg.h"
#include "qvg_kernels.cuh"
#include "qvg_ooc.hpp"
#include "qvg_plan.hpp"
#include "qvg_shard.hpp"
#include "qvg_tile_select.hpp"
#include "qvg_tile_perm.cuh"
#include "qvg_jit.hpp"

using namespace qvg;

namespace {

thread_local std::string g_last_error;

struct Status {
    int code;
    std::string msg;
};

struct CudaFail : std::runtime_error {
    int code;
    CudaFail(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return;
    // A failed call (e.g. an oversized cudaMalloc) also sets the runtime's
    // last-error slot; clear it so the next launch check does not report it.
    (void)cudaGetLastError();
    const int code = (e == cudaErrorMemoryAllocation) ? QVG_ERR_CAPACITY
                     : (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ||
                        e == cudaErrorNoKernelImageForDevice)
                         ? QVG_ERR_NO_DEVICE
                         : QVG_ERR_IO;
    throw CudaFail(code, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F> int guarded(F &&f) {
    try {
        f();
        g_last_error.clear();
        return QVG_OK;
    } catch (const CudaFail &e) {
        g_last_error = e.what();
        return e.code;
    } catch (const Validation &e) {
        g_last_error = e.what();
        return QVG_ERR_VALIDATION;
    } catch (const std::bad_alloc &) {
        g_last_error = "host allocation failed";
        return QVG_ERR_CAPACITY;
    } catch (const std::exception &e) {
        g_last_error = e.what();
        return QVG_ERR_IO;
    }
}

}  // namespace

// One rank's share of the state (or one virtual shard when several shards of
// a sharded state live on this device, see qvg_shard.hpp).
// QVG_JIT=0..3 in the environment sets the states' default QVG_OPT_JIT (0:
// the JIT passes measured no faster than k_tile overall, profiles/r02_jit_ab.json).
inline uint32_t default_jit_mode() {
    static const uint32_t m = [] {
        const char *v = std::getenv("QVG_JIT");
        return v && *v >= '0' && *v <= '3' ? (uint32_t)(*v - '0') : 0u;
    }();
    return m;
}

struct qvg_state {
    int device = 0;
    uint32_t n = 0;          // global qubits
    uint32_t L = 0;          // local qubits per shard
    uint32_t precision = 128;
    uint32_t S = 16;         // bytes per amplitude
    uint32_t rank = 0, world = 1;
    ShardSet shards;         // device buffers, transport, qubit map
    cudaStream_t stream = nullptr;
    int sm_count = 148;
    // options
    bool fuse = true;
    uint32_t tile_qubits = 11;
    uint32_t carriers = 3;
    bool low_kernel = false;   // k_pairs measured faster for targets < 5 (profiles/r01_kernel_ab.json)
    uint32_t min_run = 32;     // bytes: shortest 1-run of a forced bit that is inserted
    bool pred_store = false;   // select-and-store-all for non-inserted forced bits
    uint32_t sub_bits = 4;     // fused tile: 2^sub register amplitudes per thread (measured)
    bool fma = false;          // fused tile c128: DFMA arithmetic (not bit-identical to the reference)
    bool timing = false;       // bracket each qvg_apply with CUDA events -> stats.kernel_ms
    int exchange_mode = -1;    // QVG_OPT_EXCHANGE (-1 auto)
    int prefetch_mode = 0;     // fused tile next-tile prefetch (QVG_OPT_PREFETCH): 1 = into registers
    uint32_t batch_max = 4;    // sharded: most global qubits one exchange swaps (QVG_OPT_BATCH_EXCHANGE)
    uint32_t stage_bits = 3;   // fused tile: stage first/last group HBM access through shared memory (QVG_OPT_STAGE)
    uint32_t graph_mode = 2;   // QVG_OPT_GRAPH: 0 never, 1 capture every op list, 2 auto (default):
                               // capture an op list of >= kGraphMinOps ops the second time it is applied
    std::vector<uint64_t> graph_seen;  // auto mode: keys applied once (ring)
    uint32_t reorder = REORDER_EXACT;  // QVG_OPT_REORDER: commutation-aware fusion order (qvg_plan.hpp)
    bool classes = true;       // QVG_OPT_CLASSES: structured-matrix op bodies in fused tiles
    int tile_grid = -1;        // QVG_OPT_TILE_GRID: 0 persistent CTAs over tiles, 1 one CTA per tile, -1 auto
    uint32_t tile_order = 0;   // QVG_OPT_TILE_ORDER: 0 strided tiles per CTA, 1 contiguous chunks
    bool perm = false;         // QVG_OPT_PERM: permutation / sign-flip runs through k_tile_perm (measured
                               // equal to k_tile, profiles/r02_perm_ab.json: off by default)
    uint32_t jit_mode = default_jit_mode();  // QVG_OPT_JIT: fused passes as specialised kernels (qvg_jit.hpp); 1 async, 2 sync, 0 off
    bool capturing = false;    // run_local inside a graph capture (JIT: lookups only)
    int pipe_stages = -1;  // QVG_OPT_PIPE: -1 auto (pipe_mode below), 0 k_tile, 2/3 bulk-copy ring stages (k_tile_pipe), 4 tensor-map TMA, 5/6 k_tile_ahead (every pass / light passes)
    bool shape_set = false;    // tile_qubits / sub_bits set by the caller (no small-state default)
    struct GraphEntry {
        uint64_t key = 0;
        std::vector<qvg_gate> ops;
        cudaGraphExec_t exec = nullptr;
        qvg_stats delta{};
        uint64_t last_use = 0;
    };
    std::vector<GraphEntry> graphs;  // small LRU cache
    uint64_t graph_clock = 0;
    struct Timed {
        cudaEvent_t a, b;
        int kind;  // 0: gate passes -> kernel_ms, 1: exchange -> exchange_ms
    };
    std::vector<Timed> pending;
    qvg_step_hook_fn hook = nullptr;  // qvg_set_step_hook (tests)
    void *hook_user = nullptr;
    // device scratch
    double *d_partials = nullptr;
    double *d_probs = nullptr;
    qvg_stats stats{};
};

namespace {

constexpr int kNormBlocks = 1184;  // 8 x 148 SMs; fixed => deterministic norm
constexpr uint64_t kProbChunk = 1ull << 24;

// ------------------------------------------------------------------------
// Launchers. All grids are exact power-of-two covers of the enumeration, so
// the kernels carry no bounds checks.
// Forced bits (controls, phase targets) whose 1-runs are at least
// s.min_run bytes are inserted into the enumeration (only those amplitudes
// move); shorter runs would turn into scattered sub-granule DRAM accesses, so
// they are selected per amplitude inside a dense pass instead.
template <class R>
bool inserted(const qvg_state &s, int bit) {
    return bit >= 0 && ((uint64_t)sizeof(typename Cplx<R>::T) << bit) >= s.min_run;
}

template <class R>
void launch_pairs(const qvg_state &s, void *psi, uint32_t L, const qvg_gate &g, const OpInfo &o) {
    using T = typename Cplx<R>::T;
    Mat<R> m;
    for (int i = 0; i < 8; ++i) m.u[i] = (R)g.u[i];
    int lo = o.target, hi = -1, c_pred = -1;
    uint64_t setm = 0;
    if (inserted<R>(s, o.control)) {
        lo = std::min(o.target, o.control);
        hi = std::max(o.target, o.control);
        setm = 1ull << o.control;
    } else if (o.control >= 0) {
        c_pred = o.control;
    }
    const uint64_t npairs = 1ull << (L - 1 - (hi >= 0 ? 1 : 0));
    T *p = static_cast<T *>(psi);
    const int ps = s.pred_store ? 1 : 0;
    if (npairs >= 1024) {
        k_pairs<R, 4><<<(unsigned)(npairs / 1024), 256, 0, s.stream>>>(p, o.target, lo, hi, setm, c_pred, ps, m);
    } else {
        const unsigned bs = (unsigned)std::min<uint64_t>(npairs, 256);
        k_pairs<R, 1><<<(unsigned)(npairs / bs), bs, 0, s.stream>>>(p, o.target, lo, hi, setm, c_pred, ps, m);
    }
}

template <class R>
void launch_low(const qvg_state &s, void *psi, uint32_t L, const qvg_gate &g, const OpInfo &o) {
    using T = typename Cplx<R>::T;
    Mat<R> m;
    for (int i = 0; i < 8; ++i) m.u[i] = (R)g.u[i];
    const bool ins = inserted<R>(s, o.control);
    const int c_ins = ins ? o.control : -1;
    const int c_pred = (o.control >= 0 && !ins) ? o.control : -1;
    const int qm = 1 << ((c_ins >= 0 && c_ins < o.target) ? o.target - 1 : o.target);
    const uint64_t count = 1ull << (L - (c_ins >= 0 ? 1 : 0));
    T *p = static_cast<T *>(psi);
    if (count >= 1024) {
        k_low<R, 4><<<(unsigned)(count / 1024), 256, 0, s.stream>>>(p, o.target, qm, c_ins, c_pred, m);
    } else {
        const unsigned bs = (unsigned)std::min<uint64_t>(count, 256);
        k_low<R, 1><<<(unsigned)(count / bs), bs, 0, s.stream>>>(p, o.target, qm, c_ins, c_pred, m);
    }
}

template <class R>
void launch_phase(const qvg_state &s, void *psi, uint32_t L, const qvg_gate &g, const OpInfo &o) {
    using T = typename Cplx<R>::T;
    int bits[2] = {o.target, o.control};
    int ins[2] = {-1, -1}, nins = 0;
    uint64_t setm = 0, selm = 0;
    for (int b : bits) {
        if (b < 0) continue;
        if (inserted<R>(s, b)) {
            ins[nins++] = b;
            setm |= 1ull << b;
        } else {
            selm |= 1ull << b;
        }
    }
    if (nins == 2 && ins[0] > ins[1]) std::swap(ins[0], ins[1]);
    const uint64_t count = 1ull << (L - nins);
    T *p = static_cast<T *>(psi);
    const R dr = (R)g.u[6], di = (R)g.u[7];
    const int ps = s.pred_store ? 1 : 0;
    if (count >= 1024) {
        k_phase<R, 4><<<(unsigned)(count / 1024), 256, 0, s.stream>>>(p, ins[0], ins[1], setm, selm, ps, dr, di);
    } else {
        const unsigned bs = (unsigned)std::min<uint64_t>(count, 256);
        k_phase<R, 1><<<(unsigned)(count / bs), bs, 0, s.stream>>>(p, ins[0], ins[1], setm, selm, ps, dr, di);
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        (void)cudaGetLastError();
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// The tile of a pass as one box of a <= 5-D tensor map over the state (TileTma,
// qvg_tile.cuh): dim 0 = a 128-B row (amplitude bits 0..rb-1), then the runs
// of tile / non-tile qubits above it. False when the pass needs more than 5
// dims (it then runs k_tile).
bool tma_tile_map(const TileGeom &g, int amp_bytes, void *psi, TileTma &out) {
    // complex128 only: SWIZZLE_128B permutes 16-B chunks, which is k_tile's
    // swz() only when one amplitude is one chunk (a complex64 pass through the
    // TMA kernel measured wrong, round 2; it runs k_tile)
    if (amp_bytes != 16) return false;
    const int rb = 3;
    if (g.lowc < rb) return false;
    struct Seg { int start, len, gap; };
    std::vector<Seg> segs;
    if (g.lowc > rb) segs.push_back({rb, g.lowc - rb, 0});
    int cur = g.lowc;
    for (int i = 0; i < g.nhi;) {
        int j = i;
        while (j + 1 < g.nhi && g.hiq[j + 1] == g.hiq[j] + 1) ++j;
        const int start = g.hiq[i], len = j - i + 1;
        if (start > cur) segs.push_back({cur, start - cur, 1});
        segs.push_back({start, len, 0});
        cur = start + len;
        i = j + 1;
    }
    if (cur < g.n) segs.push_back({cur, g.n - cur, 1});
    if (segs.size() > 4) return false;
    for (const Seg &sg : segs)
        if ((!sg.gap && sg.len > 8) || sg.len > 32) return false;
    const auto encode = tensor_map_encoder();
    if (!encode) return false;
    cuuint64_t dim[5], stride[4];
    cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
    dim[0] = 16;  // 8-byte elements: one 128-B row
    box[0] = 16;
    for (int d = 1; d < 5; ++d) {
        if (d - 1 < (int)segs.size()) {
            const Seg &sg = segs[d - 1];
            dim[d] = 1ull << sg.len;
            stride[d - 1] = (cuuint64_t)amp_bytes << sg.start;
            box[d] = sg.gap ? 1u : (1u << sg.len);
            out.shift[d] = sg.start;
            out.len[d] = sg.len;
            out.gap[d] = sg.gap;
        } else {
            dim[d] = 1;
            stride[d - 1] = (cuuint64_t)amp_bytes << g.n;
            box[d] = 1;
            out.shift[d] = 0;
            out.len[d] = 0;
            out.gap[d] = 0;
        }
    }
    out.shift[0] = out.len[0] = out.gap[0] = 0;
    const CUresult r = encode(&out.map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, psi, dim, stride, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return true;
}

// A fused pass of only permutations and +-1 phases (PASS_PERM): one scatter
// through shared memory (qvg_tile_perm.cuh). 16 amplitudes per thread for the
// default tiles (2^11 complex128, 2^12 complex64), 8 for smaller ones.
template <class R>
void launch_perm(qvg_state &s, void *psi, const Pass &p, const TileOp *recs) {
    using T = typename Cplx<R>::T;
    const TileGeom &g = p.geom;
    if (g.nrec > kMaxTileRecs) throw std::runtime_error("internal: permutation pass exceeds the record limit");
    thread_local TileParams prm;
    prm.g = g;
    prm.g.order = (int)s.tile_order;
    std::memcpy(prm.ops, recs + p.op_begin, sizeof(TileOp) * g.nrec);
    const bool e16 = g.k >= (sizeof(R) == 8 ? 11 : 12);
    const unsigned threads = 1u << (g.k - (e16 ? 4 : 3));
    const size_t smem = (((sizeof(uint64_t) << g.nhi) + 15) & ~size_t(15)) + (sizeof(T) << g.k);
    const bool wide = threads > 128;
    auto kern = e16 ? (wide ? k_tile_perm<R, 16, 256> : k_tile_perm<R, 16, 128>)
                    : (wide ? k_tile_perm<R, 8, 256> : k_tile_perm<R, 8, 128>);
    static std::atomic<uint64_t> attr_set[64];  // [device]: bit per (precision, E, width)
    const uint64_t bit = 1ull << ((sizeof(R) == 8 ? 4 : 0) + (e16 ? 2 : 0) + (wide ? 1 : 0));
    std::atomic<uint64_t> &set = attr_set[s.device & 63];
    if (!(set.load(std::memory_order_acquire) & bit)) {
        cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024),
                   "cudaFuncSetAttribute(k_tile_perm)");
        set.fetch_or(bit, std::memory_order_acq_rel);
    }
    int per_sm = 0;
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (int)threads, smem), "occupancy(k_tile_perm)");
    const uint64_t grid = std::min<uint64_t>(g.ntiles, (uint64_t)std::max(per_sm, 1) * s.sm_count);
    kern<<<(unsigned)grid, threads, smem, s.stream>>>(static_cast<T *>(psi), prm);
}

// Which fused passes run as JIT kernels under QVG_OPT_JIT 1/2: those of at
// least 32 ops, three quarters of them diagonal (the QFT's controlled-phase
// passes). Their specialised kernel runs a run of same-shape phases as one
// loop over the records with no per-op dispatch: ~7% faster per heavy QFT
// pass at n = 30 (profiles/r02_jit_loop_ab.json). On passes of general,
// U3 or +-1/2 bodies the JIT kernels measured slower (spills, i-cache), so
// they keep k_tile.
bool jit_pays(const TileGeom &g, const TileOp *recs, size_t) {
    int ops = 0, diag = 0;
    for (int i = 0; i < g.nrec; ++i) {
        if (recs[i].kind == TILE_GROUP) continue;
        ++ops;
        diag += recs[i].kind == TILE_DIAG;
    }
    return ops >= 32 && 4 * diag >= 3 * ops;
}

constexpr uint32_t kJitMinQubits = 24;

// Whether a fused pass runs as a JIT kernel, and which: the plain k_tile
// variants only (no register prefetch, no bulk-copy pipelines), the passes
// jit_pays picks (QVG_OPT_JIT 1/2) or every pass (3).
bool jit_variant(const qvg_state &s, const Pass &p, const TileOp *recs, size_t amp_bytes, JitVariant *out) {
    const TileGeom &g = p.geom;
    if (!s.jit_mode || p.kind != PASS_TILE) return false;
    if (s.prefetch_mode == 1 && g.sub == 3) return false;
    const unsigned threads = 1u << (g.k - g.sub);
    if (threads == (unsigned)kPipeConsumers && s.pipe_stages >= 2 && s.pipe_stages <= 5) return false;  // an explicit pipeline
    // by default only for states whose passes outweigh a compile (~0.2-1 s per
    // kernel, once per pass structure): >= 2^24 amplitudes per shard / window
    if (s.jit_mode != 3 && (g.n < (int)kJitMinQubits || !jit_pays(g, recs, amp_bytes))) return false;
    *out = JitVariant{(int)amp_bytes, g.sub, s.fma && amp_bytes == 16, threads <= 128 ? 128 : threads <= 256 ? 256 : 512,
                      kClsSets[class_set_index(g.cls_set)]};
    return true;
}

// Compile (in parallel) the JIT kernels a plan will launch that are not
// cached yet; never inside a stream capture (apply_graph prepares first).
void jit_prepare_plan(const qvg_state &s, const Plan &plan) {
    if (!s.jit_mode || s.capturing) return;
    std::vector<JitRequest> reqs;
    for (const Pass &p : plan.passes) {
        JitVariant v{};
        if (jit_variant(s, p, plan.tile_ops.data() + p.op_begin, s.S, &v))
            reqs.push_back(JitRequest{&p.geom, plan.tile_ops.data() + p.op_begin, v, nullptr});
    }
    if (!reqs.empty()) jit_prepare(reqs.data(), reqs.size());
}

#ifdef QVG_TILE_TRACE
// Debug builds only (tools/tile_trace.py): phase stamps of the tiles
// [first, first + count) of every following k_tile launch go to `buf`.
static unsigned long long *g_trace_buf = nullptr;
static uint64_t g_trace_first = 0, g_trace_count = 0, g_trace_launches = 0, g_trace_launch = 0;
#endif

// QVG_OPT_PIPE resolved: auto = 6 (k_tile_ahead for light passes) for complex128, 0 (k_tile) for complex64,
// where the ahead kernel measured within +-3% per pass.
inline int pipe_mode(const qvg_state &s) { return s.pipe_stages >= 0 ? s.pipe_stages : (s.S == 16 ? 6 : 0); }
constexpr double kAheadMaxWeight = 300.0;
// Tiles per CTA of a "one CTA per tile" grid: up to 16 (a power of two) while at least four waves of CTAs
// remain, so CTAs still start staggered and balance uneven tiles.
constexpr uint64_t kTilesPerCta = 16;
inline uint64_t tiles_per_cta(uint64_t ntiles, uint64_t resident) {
    uint64_t t = 1;
    while (t < kTilesPerCta && ntiles / (2 * t) >= 4 * resident) t *= 2;
    return t;
}

template <class R>
void launch_tile(qvg_state &s, void *psi, const Pass &p, const TileOp *recs) {
    using T = typename Cplx<R>::T;
    const TileGeom &g = p.geom;
    if (g.nrec > kMaxTileRecs) throw std::runtime_error("internal: tile pass exceeds the record limit");
    thread_local TileParams prm;  // 25 KB; the launch copies it into the parameter block (per host thread: states on different threads may launch concurrently)
    prm.g = g;
    prm.g.order = (int)s.tile_order;
#ifdef QVG_TILE_TRACE
    prm.g.trace = g_trace_buf && g_trace_launch < g_trace_launches
                      ? g_trace_buf + 24 * g_trace_count * g_trace_launch++ : nullptr;
    prm.g.trace_first = g_trace_first;
    prm.g.trace_count = g_trace_count;
#endif
    std::memcpy(prm.ops, recs + p.op_begin, sizeof(TileOp) * g.nrec);
    unsigned threads = 1u << (g.k - g.sub);  // one 2^sub-amplitude subcube per thread
    const bool pf = s.prefetch_mode == 1 && g.sub == 3;  // register prefetch needs the 8-amplitude subcube
    size_t smem = (((sizeof(uint64_t) << g.nhi) + 15) & ~size_t(15)) +
                  (g.ngroups > 1 || g.stage ? (sizeof(T) << g.k) : 0);
    const bool fma = s.fma && sizeof(R) == 8;  // complex64 always contracts
    const bool small = threads <= 256;
    const bool tiny = threads <= 128;  // sub 4 at k <= 11: 128-thread CTAs
    // the bulk-copy pipelines serve 128-thread tiles (every default shape)
    const bool pipe_ok = threads == (unsigned)kPipeConsumers && !pf;
    const int pm = pipe_mode(s);
    const bool tma = pipe_ok && pm == 4 && tma_tile_map(g, (int)sizeof(T), psi, prm.tma);
    const int pipe = (!tma && pipe_ok && (pm == 2 || pm == 3)) ? pm : 0;
    // k_tile_ahead (qvg_tile_ahead.cuh): 16-amplitude subcubes in 128- or 256-thread CTAs; it always uses the
    // shared tile. QVG_OPT_PIPE 5: every eligible pass. 6 (auto for complex128): passes whose FP64 work per pair
    // is light enough for the hidden load to pay (tile_pass_weight <= kAheadMaxWeight; heavier passes are
    // FP64-issue bound and measured 0-8% slower, profiles/r02_ahead_ab.json) on grids with at least two tiles
    // per CTA (with one there is no next tile to load ahead).
    const uint64_t per_cta = tiles_per_cta(g.ntiles, 5ull * s.sm_count);
    const bool ahead_ok = !pf && g.sub == 4 && (threads == 128 || threads == 256);  // (32-amplitude complex64 subcubes spill there)
    const bool ahead = ahead_ok && (pm == 5 || pm == 6) && !fma &&
                       (pm == 5 || (s.tile_grid != 0 && per_cta >= 2 &&
                                    tile_pass_weight(prm.ops, g.nrec) <= kAheadMaxWeight));
    if (ahead) {
        smem = (((sizeof(uint64_t) << g.nhi) + 15) & ~size_t(15)) + (sizeof(T) << g.k);
    } else if (tma) {
        threads = kPipeThreads;
        smem = tma_smem_bytes(g.k, (int)sizeof(T), 2);
    } else if (pipe) {
        threads = kPipeThreads;
        smem = pipe_smem_bytes(g.nhi, g.k, (int)sizeof(T), pipe >= 3 ? 3 : 2);
    }
    // A JIT-specialised kernel for this pass (qvg_jit.hpp), compiled by
    // run_local's jit_prepare_plan before the apply's first launch.
    JitVariant jv{};
    if (jit_variant(s, p, prm.ops, sizeof(T), &jv)) {
        if (void *fn = jit_lookup(g, prm.ops, jv)) {
            const int per_sm = jit_occupancy(fn, threads, smem);
            const uint64_t grid = std::min<uint64_t>(g.ntiles, (uint64_t)per_sm * s.sm_count);
            cuda_check(jit_launch(fn, (unsigned)grid, threads, smem, s.stream, psi, &prm), "JIT tile launch");
            s.stats.jit_passes += 1;
            return;
        }
    }
    // Passes without structured ops (classes off) use the REAL-set kernel:
    // their records only name general bodies, which every set compiles.
    const int set_idx = class_set_index(g.cls_set);
    const TileKernel<R> kern = tile_kernel<R>(set_idx, TileVariant{g.sub, tiny, small, fma, pf, pipe, tma, ahead});
    // The shared-memory opt-in is a per-device function attribute: set it once
    // per (device, variant).
    static std::atomic<uint64_t> attr_set[64][4][16];  // [device][class set][variant / 64]: a bit per variant
    const int variant = (sizeof(R) == 8 ? 1 : 0) | (g.sub == 4 ? 2 : 0) | (fma ? 4 : 0) | (small ? 8 : 0) |
                        (pf ? 16 : 0) | (tiny ? 32 : 0) | (g.sub == 5 ? 64 : 0) | (pipe ? (pipe >= 3 ? 256 : 128) : 0) |
                        (tma ? 384 : 0) | (ahead ? 512 : 0);
    std::atomic<uint64_t> &set = attr_set[s.device & 63][set_idx][variant >> 6];
    const uint64_t bit = 1ull << (variant & 63);
    if (!(set.load(std::memory_order_acquire) & bit)) {
        cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024),
                   "cudaFuncSetAttribute(k_tile)");
        set.fetch_or(bit, std::memory_order_acq_rel);
    }
    int per_sm = 0;
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (int)threads, smem), "occupancy(k_tile)");
    per_sm = std::max(per_sm, 1);
    // persistent (one wave of CTAs looping over tiles) or a CTA per tile (QVG_OPT_TILE_GRID 1; the hardware
    // scheduler staggers CTAs, which balances passes whose work per tile varies, e.g. QFT phases controlled by a
    // qubit outside the tile). Auto = per tile: with up to 16 tiles per CTA (below) it measured faster than the
    // persistent wave in both precisions (complex128 C1 -9%, complex64 C1 -8%, C2 -5%;
    // profiles/r02_tile_grid_ab.json, r02_ahead_ab.json).
    const bool per_tile = !tma && !pipe && (s.tile_grid < 0 || s.tile_grid == 1);
    // "One CTA per tile" runs up to kTilesPerCta tiles per CTA (b, b + grid, ...) while that leaves several
    // waves of CTAs: the CTA preamble (offset table, first barrier) is paid once per 16 tiles and k_tile_ahead
    // hides 15 of 16 loads, while CTAs still start staggered and balance uneven tiles (a fully persistent
    // grid measured 9% slower for k_tile_ahead, profiles/r02_ahead_ab.json).
    const uint64_t resident = (uint64_t)per_sm * s.sm_count;
    const uint64_t split = g.ntiles / tiles_per_cta(g.ntiles, resident);
    const uint64_t grid = per_tile ? std::min<uint64_t>(split, 0x7fffffffull) : std::min<uint64_t>(g.ntiles, resident);
    kern<<<(unsigned)grid, threads, smem, s.stream>>>(static_cast<T *>(psi), prm);
}

// The engine's default tile shape for a precision (create_impl; measured in
// profiles/r01_fused_ab.json, r01_fused_ab_c64.json, r01_sub5_ab.json).
struct TileShape {
    uint32_t tile_qubits, sub_bits, carriers;
};
TileShape default_shape(uint32_t precision) {
    return precision == QVG_C128 ? TileShape{11, 4, 3} : TileShape{12, 5, 4};
}

// Small complex128 states: 2^10-amplitude tiles of 8-amplitude subcubes
// (4x the CTAs of the default 2^11 x 16 shape) unless the caller chose a
// shape. tools/tile_size_small.py, config 0's circuit: n=16 0.64-0.65 ->
// 0.57-0.61 ms on two boxes; from n=18 on the default shape is as fast or faster.
void small_state_shape(PlanOptions &po, uint32_t precision, uint32_t L, bool shape_set) {
    if (!shape_set && precision == QVG_C128 && L <= 17) {
        po.tile_qubits = std::min<uint32_t>(10, L);
        po.sub_bits = 3;
    }
}

PlanOptions plan_options(const qvg_state &s) {
    PlanOptions po;
    po.n = s.L;
    po.amp_bytes = s.S;
    po.fuse = s.fuse;
    po.tile_qubits = s.tile_qubits;
    po.carriers = s.carriers;
    po.low_kernel = s.low_kernel;
    po.min_run = s.min_run;
    po.sub_bits = s.sub_bits;
    po.stage_bits = s.stage_bits;
    po.reorder = s.reorder;
    po.classes = s.classes;
    po.perm = s.perm;
    small_state_shape(po, s.precision, s.L, s.shape_set);
    return po;
}

// Run a batch of local ops (physical local qubit indices) on one shard buffer.
void run_local(qvg_state &s, void *psi, const qvg_gate *ops, uint64_t count) {
    if (count == 0) return;
    const PlanOptions po = plan_options(s);
    const Plan plan = plan_ops(ops, count, po);
    jit_prepare_plan(s, plan);
    const bool dbl = s.precision == QVG_C128;
    for (const Pass &p : plan.passes) {
        switch (p.kind) {
        case PASS_PAIRS:
            dbl ? launch_pairs<double>(s, psi, s.L, p.op, p.info) : launch_pairs<float>(s, psi, s.L, p.op, p.info);
            break;
        case PASS_LOW:
            dbl ? launch_low<double>(s, psi, s.L, p.op, p.info) : launch_low<float>(s, psi, s.L, p.op, p.info);
            break;
        case PASS_PHASE:
            dbl ? launch_phase<double>(s, psi, s.L, p.op, p.info) : launch_phase<float>(s, psi, s.L, p.op, p.info);
            break;
        case PASS_TILE:
            dbl ? launch_tile<double>(s, psi, p, plan.tile_ops.data())
                : launch_tile<float>(s, psi, p, plan.tile_ops.data());
            s.stats.fused_passes += 1;
            break;
        case PASS_PERM:
            dbl ? launch_perm<double>(s, psi, p, plan.tile_ops.data())
                : launch_perm<float>(s, psi, p, plan.tile_ops.data());
            s.stats.fused_passes += 1;
            break;
        }
        s.stats.passes += 1;
        s.stats.kernel_launches += 1;
        s.stats.bytes_moved += p.bytes;
    }
    cuda_check(cudaGetLastError(), "kernel launch");
}

void drop_graphs(qvg_state &s) {
    for (auto &g : s.graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    s.graphs.clear();
}

// Everything the plan of an op list depends on besides the ops themselves.
uint64_t plan_signature(const qvg_state &s) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
    mix(s.fuse); mix(s.tile_qubits); mix(s.carriers); mix(s.low_kernel); mix(s.min_run); mix(s.pred_store);
    mix(s.sub_bits); mix(s.fma); mix(s.stage_bits); mix((uint64_t)s.prefetch_mode); mix(s.L); mix(s.precision);
    mix(s.reorder); mix(s.classes); mix(s.shape_set); mix(s.pipe_stages); mix(s.perm); mix(s.jit_mode); mix(s.tile_grid); mix(s.tile_order);
    return h;
}

uint64_t ops_hash(const qvg_gate *ops, uint64_t count, uint64_t seed) {
    // 8 bytes per step (an op is 80 B): a lookup key; entries also compare the bytes
    uint64_t h = seed;
    const auto *w = reinterpret_cast<const unsigned char *>(ops);
    for (uint64_t i = 0; i < count * sizeof(qvg_gate); i += 8) {
        uint64_t x;
        std::memcpy(&x, w + i, 8);
        h = (h ^ x) * 0x9e3779b97f4a7c15ull;
        h ^= h >> 29;
    }
    return h;
}

constexpr uint64_t kGraphMinOps = 8;  // auto mode: shorter lists launch a pass or two, nothing to save

qvg_stats stats_diff(const qvg_stats &a, const qvg_stats &b) {
    qvg_stats d{};
    d.passes = a.passes - b.passes;
    d.fused_passes = a.fused_passes - b.fused_passes;
    d.kernel_launches = a.kernel_launches - b.kernel_launches;
    d.bytes_moved = a.bytes_moved - b.bytes_moved;
    d.jit_passes = a.jit_passes - b.jit_passes;
    return d;
}

// Unsharded states with QVG_OPT_GRAPH: an op list seen before (same bytes,
// same plan options) replays as one captured CUDA graph; a new one is
// captured while it runs. Removes the per-pass host planning and launch
// cost that bounds small states.
bool graph_cached(const qvg_state &s, uint64_t key) {
    for (const auto &g : s.graphs)
        if (g.key == key) return true;
    return false;
}

// QVG_OPT_GRAPH auto: replay when this op list was applied before on this
// state (a repeated circuit: the bench's steps, a parameter sweep), so a
// one-shot apply never pays the capture and instantiation.
bool graph_wanted(qvg_state &s, uint64_t key, uint64_t count) {
    if (s.graph_mode == 1) return true;
    if (s.graph_mode != 2 || count < kGraphMinOps) return false;
    if (graph_cached(s, key)) return true;
    if (std::find(s.graph_seen.begin(), s.graph_seen.end(), key) != s.graph_seen.end()) return true;
    constexpr size_t kSeen = 32;
    if (s.graph_seen.size() >= kSeen) s.graph_seen.erase(s.graph_seen.begin());
    s.graph_seen.push_back(key);
    return false;
}

void apply_graph(qvg_state &s, const qvg_gate *ops, uint64_t count, uint64_t key) {
    for (auto &g : s.graphs) {
        if (g.key == key && g.ops.size() == count &&
            std::memcmp(g.ops.data(), ops, count * sizeof(qvg_gate)) == 0) {
            cuda_check(cudaGraphLaunch(g.exec, s.stream), "cudaGraphLaunch");
            s.stats.passes += g.delta.passes;
            s.stats.fused_passes += g.delta.fused_passes;
            s.stats.kernel_launches += g.delta.kernel_launches;
            s.stats.bytes_moved += g.delta.bytes_moved;
            s.stats.jit_passes += g.delta.jit_passes;
            s.stats.graph_replays += 1;
            g.last_use = ++s.graph_clock;
            return;
        }
    }
    const qvg_stats before = s.stats;
    cudaGraph_t graph = nullptr;
    jit_prepare_plan(s, plan_ops(ops, count, plan_options(s)));  // compiles and module loads stay outside the capture
    cuda_check(cudaStreamBeginCapture(s.stream, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    s.capturing = true;
    try {
        run_local(s, s.shards.bufs[0], ops, count);
    } catch (...) {
        s.capturing = false;
        cudaStreamEndCapture(s.stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        s.stats = before;
        throw;
    }
    s.capturing = false;
    cuda_check(cudaStreamEndCapture(s.stream, &graph), "cudaStreamEndCapture");
    qvg_state::GraphEntry e;
    e.key = key;
    e.ops.assign(ops, ops + count);
    e.delta = stats_diff(s.stats, before);
    e.last_use = ++s.graph_clock;
    const cudaError_t inst = cudaGraphInstantiate(&e.exec, graph, 0);
    cudaGraphDestroy(graph);
    cuda_check(inst, "cudaGraphInstantiate");
    cuda_check(cudaGraphLaunch(e.exec, s.stream), "cudaGraphLaunch");
    s.stats.graph_replays += 1;
    constexpr size_t kMaxGraphs = 8;
    if (s.graphs.size() >= kMaxGraphs) {
        auto lru = std::min_element(s.graphs.begin(), s.graphs.end(),
                                    [](const auto &a, const auto &b) { return a.last_use < b.last_use; });
        cudaGraphExecDestroy(lru->exec);
        s.graphs.erase(lru);
    }
    s.graphs.push_back(std::move(e));
}

void set_device(const qvg_state *s) { cuda_check(cudaSetDevice(s->device), "cudaSetDevice"); }

void check_state(const qvg_state *s) {
    if (!s) throw Validation("null state");
}

void check_range(const qvg_state *s, uint64_t offset, uint64_t count) {
    const uint64_t dim = 1ull << s->n;
    if (offset > dim || count > dim - offset)
        throw Validation("amplitude range [" + std::to_string(offset) + ", " + std::to_string(offset + count) +
                         ") out of range for " + std::to_string(dim) + " amplitudes");
}

}  // namespace

// ---------------------------------------------------------------------------
// Shard executor hooks used by qvg_shard.hpp.
namespace qvg {
void cuda_throw(cudaError_t e, const char *what) { cuda_check(e, what); }
void shard_run_local(qvg_state &s, void *psi, const qvg_gate *ops, uint64_t count) { run_local(s, psi, ops, count); }
cudaStream_t shard_stream(qvg_state &s) { return s.stream; }
uint32_t shard_amp_bytes(const qvg_state &s) { return s.S; }
qvg_stats &shard_stats(qvg_state &s) { return s.stats; }
int shard_exchange_mode(const qvg_state &s) { return s.exchange_mode; }
bool shard_timing(const qvg_state &s) { return s.timing; }
void shard_time_push(qvg_state &s, cudaEvent_t a, cudaEvent_t b, int kind) { s.pending.push_back({a, b, kind}); }
bool shard_has_hook(const qvg_state &s) { return s.hook != nullptr; }
int shard_step_hook(qvg_state &s, uint32_t rank, uint64_t segment, uint32_t type, uint32_t phase) {
    return s.hook ? s.hook(s.hook_user, rank, segment, type, phase) : 0;
}
uint32_t shard_batch_max(const qvg_state &s) { return s.batch_max; }
}  // namespace qvg

extern "C" {

int qvg_abi_version(void) { return QVG_ABI_VERSION; }

const char *qvg_last_error(void) { return g_last_error.c_str(); }

static int create_impl(uint32_t n, uint32_t precision, int device, uint32_t rank, uint32_t world,
                       const void *nccl_id, bool virtual_shards, qvg_state **out) {
    return guarded([&] {
        if (!out) throw Validation("null output pointer");
        *out = nullptr;
        if (precision != QVG_C64 && precision != QVG_C128)
            throw Validation("precision must be 64 (complex64) or 128 (complex128)");
        if (world == 0 || (world & (world - 1)) != 0) throw Validation("world size must be a power of two");
        if (rank >= world) throw Validation("rank out of range");
        uint32_t g = 0;
        while ((1u << g) < world) ++g;
        if (n < 1 || n > 40) throw Validation("n_qubits must be in [1, 40]");
        if (n < g + 2 && world > 1) throw Validation("too few qubits for this many shards");
        int ndev = 0;
        cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (device < 0 || device >= ndev) throw CudaFail(QVG_ERR_NO_DEVICE, "no CUDA device " + std::to_string(device));
        auto *s = new qvg_state();
        s->device = device;
        s->n = n;
        s->L = n - g;
        s->precision = precision;
        s->S = precision == QVG_C128 ? 16 : 8;
        s->rank = rank;
        s->world = world;
        // Measured best tile shapes (profiles/r01_fused_ab.json, r01_fused_ab_c64.json,
        // r01_sub5_ab.json): complex128: 2^11 amplitudes as 128 threads x 16 register
        // amplitudes (C2/C1/C3 4-11% faster than 256 x 8); complex64: 2^12 as
        // 128 threads x 32 (C2 -16%, C1 -12% against 256 x 16, C3 +1%).
        const TileShape shape = default_shape(precision);
        s->tile_qubits = shape.tile_qubits;
        s->sub_bits = shape.sub_bits;
        s->carriers = shape.carriers;
        try {
            set_device(s);
            cuda_check(cudaDeviceGetAttribute(&s->sm_count, cudaDevAttrMultiProcessorCount, device), "sm count");
            cuda_check(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking), "cudaStreamCreate");
            cuda_check(cudaMalloc(&s->d_partials, 2 * kNormBlocks * sizeof(double)), "cudaMalloc(partials)");
            s->shards.init(*s, n, s->L, rank, world, nccl_id, virtual_shards);
            shard_init_basis(*s, s->shards, 0);
            cuda_check(cudaStreamSynchronize(s->stream), "init sync");
        } catch (...) {
            s->shards.release();
            if (s->d_partials) cudaFree(s->d_partials);
            if (s->stream) cudaStreamDestroy(s->stream);
            delete s;
            throw;
        }
        *out = s;
    });
}

int qvg_create(uint32_t n_qubits, uint32_t precision, int device, qvg_state **out) {
    return create_impl(n_qubits, precision, device, 0, 1, nullptr, false, out);
}

int qvg_create_sharded(uint32_t n_qubits, uint32_t precision, int device, uint32_t rank, uint32_t world,
                       const void *nccl_id, qvg_state **out) {
    // nccl_id == NULL: all `world` shards live on this device in one process
    // (virtual shards; exchanges are device copies). Used to test the sharded
    // path bit-for-bit on one GPU.
    return create_impl(n_qubits, precision, device, nccl_id ? rank : 0, world, nccl_id, nccl_id == nullptr, out);
}

int qvg_nccl_unique_id(void *out128) {
    return guarded([&] {
        if (!out128) throw Validation("null output pointer");
        shard_nccl_unique_id(out128);
    });
}

int qvg_destroy(qvg_state *s) {
    return guarded([&] {
        if (!s) return;
        cudaSetDevice(s->device);
        if (s->stream) cudaStreamSynchronize(s->stream);
        for (auto &pr : s->pending) {
            cudaEventDestroy(pr.a);
            cudaEventDestroy(pr.b);
        }
        drop_graphs(*s);
        s->shards.release();
        if (s->d_partials) cudaFree(s->d_partials);
        if (s->d_probs) cudaFree(s->d_probs);
        if (s->stream) cudaStreamDestroy(s->stream);
        delete s;
    });
}

int qvg_info(const qvg_state *s, uint32_t *n, uint32_t *precision, uint32_t *rank, uint32_t *world) {
    return guarded([&] {
        check_state(s);
        if (n) *n = s->n;
        if (precision) *precision = s->precision;
        if (rank) *rank = s->rank;
        if (world) *world = s->world;
    });
}

#ifdef QVG_TILE_TRACE
extern "C" void qvg_debug_tile_trace(void *buf, uint64_t first, uint64_t count, uint64_t launches) {
    g_trace_buf = static_cast<unsigned long long *>(buf);  // 24 * count * launches words
    g_trace_first = first;
    g_trace_count = count;
    g_trace_launches = launches;
    g_trace_launch = 0;
}
#endif

int qvg_set_option(qvg_state *s, int key, int64_t value) {
    return guarded([&] {
        check_state(s);
        switch (key) {
        case QVG_OPT_FUSE: s->fuse = value != 0; break;
        case QVG_OPT_TILE_QUBITS: {
            const int64_t maxk = 12;  // k_tile runs 2^(k-3) <= 512 threads
            if (value < 2 || value > maxk) throw Validation("tile_qubits out of range");
            s->tile_qubits = (uint32_t)value;
            s->shape_set = true;
            break;
        }
        case QVG_OPT_CARRIERS:
            if (value < 0 || value > 10) throw Validation("carriers out of range");
            s->carriers = (uint32_t)value;
            break;
        case QVG_OPT_LOW_KERNEL: s->low_kernel = value != 0; break;
        case QVG_OPT_MIN_RUN:
            if (value < 8 || value > (1 << 20) || (value & (value - 1))) throw Validation("min_run must be a power of two >= 8");
            s->min_run = (uint32_t)value;
            break;
        case QVG_OPT_PRED_STORE: s->pred_store = value != 0; break;
        case QVG_OPT_SUB_BITS:
            if (value < 3 || value > (s->precision == QVG_C64 ? 5 : 4))
                throw Validation("sub_bits must be 3 or 4 (complex64: 3..5)");
            s->sub_bits = (uint32_t)value;
            s->shape_set = true;
            break;
        case QVG_OPT_FMA: s->fma = value != 0; break;
        case QVG_OPT_TIMING: s->timing = value != 0; break;
        case QVG_OPT_PREFETCH:
            if (value < 0 || value > 1) throw Validation("prefetch must be 0 or 1");
            s->prefetch_mode = (int)value;
            break;
        case QVG_OPT_REORDER:
            if (value < 0 || value > 2) throw Validation("reorder must be 0 (never), 1 (any commuting move) or 2 (bit-exact moves)");
            s->reorder = (uint32_t)value;
            break;
        case QVG_OPT_CLASSES: s->classes = value != 0; break;
        case QVG_OPT_GRAPH:
            if (value < 0 || value > 2) throw Validation("graph must be 0 (never), 1 (always) or 2 (auto)");
            s->graph_mode = (uint32_t)value;
            if (!s->graph_mode) drop_graphs(*s);
            s->graph_seen.clear();
            break;
        case QVG_OPT_STAGE:
            if (value < 0 || value > 12) throw Validation("stage must be 0 (never) .. 12");
            s->stage_bits = (uint32_t)value;
            break;
        case QVG_OPT_BATCH_EXCHANGE:
            if (value < 1 || value > 4) throw Validation("batch exchange must be 1..4 global qubits");
            s->batch_max = (uint32_t)value;
            break;
        case QVG_OPT_EXCHANGE:
            if (value < -1 || value > 2) throw Validation("exchange mode must be -1, 0, 1 or 2");
            s->exchange_mode = (int)value;
            break;
        case QVG_OPT_PERM: s->perm = value != 0; break;
        case QVG_OPT_TILE_GRID:
            if (value < -1 || value > 1) throw Validation("tile grid must be -1 (auto), 0 (persistent) or 1 (CTA per tile)");
            s->tile_grid = (int)value;
            break;
        case QVG_OPT_TILE_ORDER:
            if (value < 0 || value > 1) throw Validation("tile order must be 0 (strided) or 1 (contiguous per CTA)");
            s->tile_order = (uint32_t)value;
            break;
        case QVG_OPT_JIT:
            if (value < 0 || value > 3)
                throw Validation("jit must be 0 (never), 1 (async), 2 (compile before launch) or 3 (every pass, compiled first)");
            s->jit_mode = (uint32_t)value;
            break;
        case QVG_OPT_PIPE:
            if (value < -1 || value > 6 || value == 1)
                throw Validation("pipe must be 0 (k_tile), 2 or 3 (bulk-copy ring stages), 4 (tensor-map TMA), 5 (next tile's "
                                 "load under the last group, every pass) or 6 (the same for light passes)");
            s->pipe_stages = (int)value;
            break;
        case QVG_OPT_XCHG_CHUNK:
            if (value < 0 || (value % 16) != 0) throw Validation("exchange chunk must be a multiple of 16 bytes (0 = default)");
            s->shards.chunk_override = (uint64_t)value;
            break;
        default: throw Validation("unknown option " + std::to_string(key));
        }
    });
}

int qvg_init_basis(qvg_state *s, uint64_t index) {
    return guarded([&] {
        check_state(s);
        if (index >= (1ull << s->n)) throw Validation("basis index out of range");
        set_device(s);
        shard_init_basis(*s, s->shards, index);
        cuda_check(cudaStreamSynchronize(s->stream), "init_basis");
    });
}

int qvg_load(qvg_state *s, const void *host, uint64_t offset, uint64_t count) {
    return guarded([&] {
        check_state(s);
        check_range(s, offset, count);
        if (count && !host) throw Validation("null host buffer");
        set_device(s);
        shard_transfer(*s, s->shards, const_cast<void *>(host), offset, count, true);
    });
}

int qvg_read(qvg_state *s, void *host, uint64_t offset, uint64_t count) {
    return guarded([&] {
        check_state(s);
        check_range(s, offset, count);
        if (count && !host) throw Validation("null host buffer");
        set_device(s);
        shard_transfer(*s, s->shards, host, offset, count, false);
    });
}

int qvg_host_alloc(uint64_t bytes, void **out) {
    return guarded([&] {
        if (!out) throw Validation("null output pointer");
        *out = nullptr;
        cuda_check(cudaHostAlloc(out, bytes, cudaHostAllocPortable), "cudaHostAlloc");
    });
}

int qvg_host_free(void *ptr) {
    return guarded([&] {
        if (ptr) cuda_check(cudaFreeHost(ptr), "cudaFreeHost");
    });
}

int qvg_load_async(qvg_state *s, const void *host, uint64_t offset, uint64_t count) {
    return guarded([&] {
        check_state(s);
        check_range(s, offset, count);
        if (count && !host) throw Validation("null host buffer");
        set_device(s);
        shard_transfer(*s, s->shards, const_cast<void *>(host), offset, count, true, false);
    });
}

int qvg_read_async(qvg_state *s, void *host, uint64_t offset, uint64_t count) {
    return guarded([&] {
        check_state(s);
        check_range(s, offset, count);
        if (count && !host) throw Validation("null host buffer");
        set_device(s);
        shard_transfer(*s, s->shards, host, offset, count, false, false);
    });
}

int qvg_apply(qvg_state *s, const qvg_gate *ops, uint64_t count) {
    return guarded([&] {
        check_state(s);
        if (count && !ops) throw Validation("null op array");
        for (uint64_t i = 0; i < count; ++i) validate_op(ops[i], s->n, i);
        set_device(s);
        nvtxRangePushA("qvg_apply");
        // Timing: an unsharded apply is one bracketed interval (kernel_ms); a
        // sharded one is timed per segment inside the executor (local passes
        // -> kernel_ms, exchanges -> exchange_ms, qvg_shard.hpp run_steps).
        const bool whole = s->timing && s->world == 1;
        cudaEvent_t ev[2] = {nullptr, nullptr};
        if (whole) {
            for (auto &e : ev) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
            cuda_check(cudaEventRecord(ev[0], s->stream), "cudaEventRecord");
        }
        uint64_t key = 0;
        const bool graph = s->world == 1 && count > 0 && s->graph_mode &&
                           graph_wanted(*s, key = ops_hash(ops, count, plan_signature(*s)), count);
        if (graph) apply_graph(*s, ops, count, key);
        else shard_apply(*s, s->shards, ops, count);
        if (whole) {
            cuda_check(cudaEventRecord(ev[1], s->stream), "cudaEventRecord");
            s->pending.push_back({ev[0], ev[1], 0});
        }
        nvtxRangePop();
        s->stats.gates_applied += count;
    });
}

int qvg_sync(qvg_state *s) {
    return guarded([&] {
        check_state(s);
        set_device(s);
        cuda_check(cudaStreamSynchronize(s->stream), "cudaStreamSynchronize");
        shard_check_async(s->shards);  // NCCL errors surface as IoError
    });
}

int qvg_norm(qvg_state *s, double *out) {
    return guarded([&] {
        check_state(s);
        if (!out) throw Validation("null output pointer");
        set_device(s);
        std::vector<double> partial(kNormBlocks);
        double sum = 0.0, carry = 0.0;
        auto kahan = [&](double term) {
            const double t = term - carry;
            const double next = sum + t;
            carry = (next - sum) - t;
            sum = next;
        };
        const uint64_t local = 1ull << s->L;
        for (void *psi : s->shards.local_buffers()) {
            if (s->precision == QVG_C128)
                k_norm_partials<double><<<kNormBlocks, 256, 0, s->stream>>>(static_cast<const double2 *>(psi), local,
                                                                            s->d_partials);
            else
                k_norm_partials<float><<<kNormBlocks, 256, 0, s->stream>>>(static_cast<const float2 *>(psi), local,
                                                                           s->d_partials);
            cuda_check(cudaGetLastError(), "norm launch");
            cuda_check(cudaMemcpyAsync(partial.data(), s->d_partials, kNormBlocks * sizeof(double),
                                       cudaMemcpyDeviceToHost, s->stream),
                       "norm D2H");
            cuda_check(cudaStreamSynchronize(s->stream), "norm sync");
            for (double v : partial) kahan(v);
        }
        sum = shard_allreduce_sum(*s, s->shards, sum);
        *out = std::sqrt(sum);
    });
}

int qvg_probabilities(qvg_state *s, double *out, uint64_t offset, uint64_t count) {
    return guarded([&] {
        check_state(s);
        check_range(s, offset, count);
        if (count && !out) throw Validation("null output pointer");
        set_device(s);
        shard_canonicalize(*s, s->shards);
        if (!s->d_probs) cuda_check(cudaMalloc(&s->d_probs, kProbChunk * sizeof(double)), "cudaMalloc(probs)");
        // Each rank fills the part of [offset, offset+count) it owns; the
        // rest of `out` is left untouched (gather is the caller's job).
        const uint64_t local = 1ull << s->L;
        const std::vector<void *> bufs = s->shards.local_buffers();
        const std::vector<uint32_t> ranks = s->shards.local_ranks();
        for (size_t b = 0; b < bufs.size(); ++b) {
            const uint64_t lo = (uint64_t)ranks[b] * local, hi = lo + local;
            const uint64_t a = std::max(lo, offset), e = std::min(hi, offset + count);
            for (uint64_t x = a; x < e; x += kProbChunk) {
                const uint64_t c = std::min(kProbChunk, e - x);
                const unsigned grid = (unsigned)std::min<uint64_t>((c + 255) / 256, 4096);
                if (s->precision == QVG_C128)
                    k_probs<double><<<grid, 256, 0, s->stream>>>(static_cast<const double2 *>(bufs[b]) + (x - lo), c,
                                                                 s->d_probs);
                else
                    k_probs<float><<<grid, 256, 0, s->stream>>>(static_cast<const float2 *>(bufs[b]) + (x - lo), c,
                                                                s->d_probs);
                cuda_check(cudaGetLastError(), "probs launch");
                cuda_check(cudaMemcpyAsync(out + (x - offset), s->d_probs, c * sizeof(double), cudaMemcpyDeviceToHost,
                                           s->stream),
                           "probs D2H");
            }
        }
        cuda_check(cudaStreamSynchronize(s->stream), "probs sync");
    });
}

int qvg_top_amplitudes(qvg_state *s, uint32_t k, uint64_t *index_out, double *amps_out) {
    return guarded([&] {
        check_state(s);
        if (k && (!index_out || !amps_out)) throw Validation("null output pointer");
        set_device(s);
        shard_top_amplitudes(*s, s->shards, k, index_out, amps_out);
    });
}

}  // extern "C"

static void check_same_shape(const qvg_state *a, const qvg_state *b) {
    if (!a || !b) throw Validation("null state");
    if (a->n != b->n || a->precision != b->precision || a->world != b->world || a->rank != b->rank ||
        a->device != b->device || a->shards.is_virtual != b->shards.is_virtual)
        throw Validation("states differ in shape (qubits, precision, sharding or device)");
}

// Two-state reduction over matching local shard buffers; both states are
// first brought to canonical order and `b`'s work is ordered before `a`'s
// stream reads it.
template <class Launch>
static void two_state_reduce(qvg_state *a, qvg_state *b, int words, Launch launch, std::vector<double> &partials) {
    check_same_shape(a, b);
    set_device(a);
    shard_canonicalize(*a, a->shards);
    shard_canonicalize(*b, b->shards);
    cuda_check(cudaStreamSynchronize(b->stream), "sync second state");
    const uint64_t local = 1ull << a->L;
    const std::vector<void *> pa = a->shards.local_buffers(), pb = b->shards.local_buffers();
    partials.assign((size_t)kNormBlocks * words * pa.size(), 0.0);
    for (size_t i = 0; i < pa.size(); ++i) {
        launch(pa[i], pb[i], local);
        cuda_check(cudaGetLastError(), "reduction launch");
        cuda_check(cudaMemcpyAsync(partials.data() + (size_t)kNormBlocks * words * i, a->d_partials,
                                   (size_t)kNormBlocks * words * sizeof(double), cudaMemcpyDeviceToHost, a->stream),
                   "D2H partials");
        cuda_check(cudaStreamSynchronize(a->stream), "reduction sync");
    }
}

extern "C" {

int qvg_inner_product(qvg_state *a, qvg_state *b, double *re, double *im) {
    return guarded([&] {
        if (!re || !im) throw Validation("null output pointer");
        std::vector<double> part;
        two_state_reduce(a, b, 2, [&](void *x, void *y, uint64_t local) {
            if (a->precision == QVG_C128)
                k_inner_partials<double><<<kNormBlocks, 256, 0, a->stream>>>(static_cast<const double2 *>(x),
                                                                              static_cast<const double2 *>(y), local,
                                                                              a->d_partials);
            else
                k_inner_partials<float><<<kNormBlocks, 256, 0, a->stream>>>(static_cast<const float2 *>(x),
                                                                             static_cast<const float2 *>(y), local,
                                                                             a->d_partials);
        }, part);
        double sr = 0.0, cr = 0.0, si = 0.0, ci = 0.0;  // Kahan, fixed order
        for (size_t i = 0; i < part.size(); i += 2) {
            const double tr = part[i] - cr, nr = sr + tr;
            cr = (nr - sr) - tr;
            sr = nr;
            const double ti = part[i + 1] - ci, ni = si + ti;
            ci = (ni - si) - ti;
            si = ni;
        }
        *re = shard_allreduce_sum(*a, a->shards, sr);
        *im = shard_allreduce_sum(*a, a->shards, si);
    });
}

int qvg_max_deviation(qvg_state *a, qvg_state *b, double *out) {
    return guarded([&] {
        if (!out) throw Validation("null output pointer");
        std::vector<double> part;
        two_state_reduce(a, b, 1, [&](void *x, void *y, uint64_t local) {
            if (a->precision == QVG_C128)
                k_maxdiff_partials<double><<<kNormBlocks, 256, 0, a->stream>>>(static_cast<const double2 *>(x),
                                                                                static_cast<const double2 *>(y),
                                                                                local, a->d_partials);
            else
                k_maxdiff_partials<float><<<kNormBlocks, 256, 0, a->stream>>>(static_cast<const float2 *>(x),
                                                                               static_cast<const float2 *>(y),
                                                                               local, a->d_partials);
        }, part);
        double m = 0.0;
        for (double v : part)
            if (v > m || v != v) m = v;
        *out = shard_allreduce_max(*a, a->shards, m);
    });
}

int qvg_checksums(qvg_state *s, uint64_t chunk_amps, uint64_t *out, uint64_t cap, uint64_t *count) {
    return guarded([&] {
        check_state(s);
        const uint64_t dim = 1ull << s->n;
        if (chunk_amps < 4096 || (chunk_amps & (chunk_amps - 1)) || chunk_amps > dim)
            throw Validation("chunk_amps must be a power of two in [4096, 2^n]");
        const uint64_t nchunks = dim / chunk_amps;
        if (count) *count = nchunks;
        if (!out) return;
        if (cap < nchunks) throw Validation("output too small: need 2 words per chunk");
        set_device(s);
        shard_canonicalize(*s, s->shards);
        int cbits = 0;
        while ((1ull << cbits) < chunk_amps) ++cbits;
        unsigned long long *d = nullptr;
        cuda_check(cudaMalloc(&d, nchunks * 2 * sizeof(uint64_t)), "cudaMalloc(checksums)");
        std::unique_ptr<void, cudaError_t (*)(void *)> guard(d, cudaFree);
        cuda_check(cudaMemsetAsync(d, 0, nchunks * 2 * sizeof(uint64_t), s->stream), "memset checksums");
        const uint64_t local = 1ull << s->L;
        const std::vector<void *> bufs = s->shards.local_buffers();
        const std::vector<uint32_t> ranks = s->shards.local_ranks();
        for (size_t b = 0; b < bufs.size(); ++b) {
            const unsigned blocks = (unsigned)((local + 4095) / 4096);
            const uint64_t base = (uint64_t)ranks[b] * local;
            if (s->precision == QVG_C128)
                k_checksum<double><<<blocks, 256, 0, s->stream>>>(static_cast<const double2 *>(bufs[b]), local, base,
                                                                 cbits, d);
            else
                k_checksum<float><<<blocks, 256, 0, s->stream>>>(static_cast<const float2 *>(bufs[b]), local, base,
                                                                cbits, d);
            cuda_check(cudaGetLastError(), "checksum launch");
        }
        if (s->shards.comm)
            nccl_check(ncclAllReduce(d, d, nchunks * 2, ncclUint64, ncclSum, s->shards.comm, s->stream),
                       "ncclAllReduce(checksums)");
        cuda_check(cudaMemcpyAsync(out, d, nchunks * 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s->stream),
                   "D2H checksums");
        cuda_check(cudaStreamSynchronize(s->stream), "checksum sync");
    });
}

int qvg_stats_get(const qvg_state *s, qvg_stats *out) {
    return guarded([&] {
        check_state(s);
        if (!out) throw Validation("null output pointer");
        // Fold finished timed applies (QVG_OPT_TIMING) into kernel_ms; this
        // waits for the work the events bracket.
        auto *m = const_cast<qvg_state *>(s);
        for (auto &pr : m->pending) {
            float ms = 0.f;
            cuda_check(cudaEventSynchronize(pr.b), "cudaEventSynchronize");
            cuda_check(cudaEventElapsedTime(&ms, pr.a, pr.b), "cudaEventElapsedTime");
            (pr.kind ? m->stats.exchange_ms : m->stats.kernel_ms) += ms;
            cudaEventDestroy(pr.a);
            cudaEventDestroy(pr.b);
        }
        m->pending.clear();
        *out = s->stats;
    });
}

int qvg_stats_reset(qvg_state *s) {
    return guarded([&] {
        check_state(s);
        s->stats = qvg_stats{};
    });
}

int qvg_stream(const qvg_state *s, void **stream_out) {
    return guarded([&] {
        check_state(s);
        if (!stream_out) throw Validation("null output pointer");
        *stream_out = (void *)s->stream;
    });
}

int qvg_device_buffer(const qvg_state *s, void **ptr_out, uint64_t *bytes_out) {
    return guarded([&] {
        check_state(s);
        const std::vector<void *> bufs = const_cast<qvg_state *>(s)->shards.local_buffers();
        if (ptr_out) *ptr_out = bufs.empty() ? nullptr : bufs[0];
        if (bytes_out) *bytes_out = (uint64_t)s->S << s->L;
    });
}

}  // extern "C"

namespace {

// Where the out-of-core state lives. A chunk is npieces pieces of `piece`
// amplitudes at host offsets base_off + offhi[m]; window slot m holds piece m.
struct OocIo {
    virtual ~OocIo() = default;
    // enqueue (or perform) the host -> window copies of chunk c on window w
    virtual void fetch(qvg_state &W, int w, char *win, uint64_t base_off, const std::vector<uint64_t> &offhi,
                       uint64_t piece) = 0;
    // enqueue the window -> host copies
    virtual void store(qvg_state &W, int w, const char *win, uint64_t base_off, const std::vector<uint64_t> &offhi,
                       uint64_t piece) = 0;
    // all chunks of the segment are home (streams synchronized)
    virtual void drain() {}
    // true: copies are plain stream-ordered cudaMemcpyAsync, so the next
    // segment may start fetching pieces whose sources are already home
    // (fetch_piece), without a segment barrier
    virtual bool overlap_ok() const { return false; }
    virtual void fetch_piece(qvg_state &, char *, uint64_t, uint64_t, uint64_t) {}
};

// Host memory: copies go straight between the user's buffer and HBM.
struct HostMemIo : OocIo {
    char *h;
    uint64_t S;
    HostMemIo(void *host, uint64_t s) : h(static_cast<char *>(host)), S(s) {}
    void fetch(qvg_state &W, int, char *win, uint64_t base_off, const std::vector<uint64_t> &offhi,
               uint64_t piece) override {
        for (size_t m = 0; m < offhi.size(); ++m)
            cuda_check(cudaMemcpyAsync(win + m * piece * S, h + (base_off + offhi[m]) * S, piece * S,
                                       cudaMemcpyHostToDevice, W.stream),
                       "out-of-core H2D");
    }
    void store(qvg_state &W, int, const char *win, uint64_t base_off, const std::vector<uint64_t> &offhi,
               uint64_t piece) override {
        for (size_t m = 0; m < offhi.size(); ++m)
            cuda_check(cudaMemcpyAsync(h + (base_off + offhi[m]) * S, win + m * piece * S, piece * S,
                                       cudaMemcpyDeviceToHost, W.stream),
                       "out-of-core D2H");
    }
    bool overlap_ok() const override { return true; }
    // window slot `slot` <- host amplitudes [host_off, host_off + piece)
    void fetch_piece(qvg_state &W, char *win, uint64_t slot, uint64_t host_off, uint64_t piece) override {
        cuda_check(cudaMemcpyAsync(win + slot * piece * S, h + host_off * S, piece * S, cudaMemcpyHostToDevice,
                                   W.stream),
                   "out-of-core H2D");
    }
};

// Caller I/O (e.g. pread/pwrite on a QVSV file): each window has a pinned
// staging buffer; the host reads the next chunk and writes back the previous
// one while the device works on the other window.
struct CallbackIo : OocIo {
    qvg_io_fn io;
    void *user;
    uint64_t S;
    void *stage[2] = {nullptr, nullptr};
    struct Pending {
        bool live = false;
        uint64_t base_off = 0, piece = 0;
        std::vector<uint64_t> offhi;
    } pending[2];
    qvg_state *wins[2] = {nullptr, nullptr};
    CallbackIo(qvg_io_fn f, void *u, uint64_t s, uint64_t window_bytes) : io(f), user(u), S(s) {
        for (auto &p : stage) cuda_check(cudaHostAlloc(&p, window_bytes, cudaHostAllocPortable), "cudaHostAlloc(staging)");
    }
    ~CallbackIo() override {
        for (auto *p : stage)
            if (p) cudaFreeHost(p);
    }
    void call(uint64_t off, uint64_t cnt, void *buf, int write) {
        if (io(user, off, cnt, buf, write) != 0)
            throw CudaFail(QVG_ERR_IO, std::string("state I/O callback failed (") + (write ? "write" : "read") + ")");
    }
    void flush(int w) {
        if (!pending[w].live) return;
        char *st = static_cast<char *>(stage[w]);
        for (size_t m = 0; m < pending[w].offhi.size(); ++m)
            call(pending[w].base_off + pending[w].offhi[m], pending[w].piece, st + m * pending[w].piece * S, 1);
        pending[w].live = false;
    }
    void fetch(qvg_state &W, int w, char *win, uint64_t base_off, const std::vector<uint64_t> &offhi,
               uint64_t piece) override {
        wins[w] = &W;
        cuda_check(cudaStreamSynchronize(W.stream), "out-of-core staging sync");  // staging free again
        flush(w);
        char *st = static_cast<char *>(stage[w]);
        for (size_t m = 0; m < offhi.size(); ++m) call(base_off + offhi[m], piece, st + m * piece * S, 0);
        cuda_check(cudaMemcpyAsync(win, st, offhi.size() * piece * S, cudaMemcpyHostToDevice, W.stream),
                   "out-of-core H2D");
    }
    void store(qvg_state &W, int w, const char *win, uint64_t base_off, const std::vector<uint64_t> &offhi,
               uint64_t piece) override {
        cuda_check(cudaMemcpyAsync(stage[w], win, offhi.size() * piece * S, cudaMemcpyDeviceToHost, W.stream),
                   "out-of-core D2H");
        pending[w] = Pending{true, base_off, piece, offhi};
    }
    void drain() override {
        for (int w = 0; w < 2; ++w) flush(w);
    }
};

// The out-of-core executor shared by qvg_apply_host and qvg_apply_stream.
// Chunks rotate over `nwin` device windows, each on its own stream, so chunk
// k+1's H2D and gates overlap chunk k's D2H. Between segments (the qubit
// grouping changes, so every new chunk gathers pieces of every old one):
//   * overlap-capable I/O (host memory): no barrier. Each piece of a new chunk
//     waits only for the D2H event of the LAST old chunk it overlaps, and the
//     pieces are fetched in the order their sources come home, so the first
//     chunk of segment s+1 loads while the last chunks of segment s drain;
//   * caller I/O (file callbacks through staging buffers): a full barrier.
void ooc_run(OocIo &io, uint32_t n, uint32_t precision, uint32_t w, const qvg_gate *ops, uint64_t count,
             qvg_state *const *win, int nwin, qvg_stats *stats_out) {
    const uint64_t S = precision == QVG_C128 ? 16 : 8;
    const std::vector<OocSegment> segs = plan_ooc(n, w, ops, count);
    std::vector<qvg_gate> local;
    uint64_t host_bytes = 0;
    const uint64_t nchunks = 1ull << (n - w);
    std::vector<cudaEvent_t> done[2];  // D2H-complete event per chunk: previous / current segment
    for (auto &v : done) {
        v.assign(nchunks, nullptr);
        for (auto &e : v) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    }
    struct EvFree {
        std::vector<cudaEvent_t> *d;
        ~EvFree() {
            for (int i = 0; i < 2; ++i)
                for (auto e : d[i]) cudaEventDestroy(e);
        }
    } ev_free{done};
    const bool overlap = io.overlap_ok();
    uint64_t seq = 0;  // chunk sequence number across segments: window = seq % nwin
    const OocSegment *prev = nullptr;
    std::vector<uint64_t> order;
    std::vector<uint64_t> dep;
    for (const OocSegment &sg : segs) {
        const uint64_t piece = 1ull << sg.lowc;
        const uint64_t npieces = 1ull << sg.hiq.size();
        std::vector<uint64_t> offhi(npieces, 0);
        for (uint64_t m = 0; m < npieces; ++m)
            for (size_t b = 0; b < sg.hiq.size(); ++b)
                if ((m >> b) & 1) offhi[m] |= 1ull << sg.hiq[b];
        for (uint64_t c = 0; c < nchunks; ++c, ++seq) {
            const int wi = (int)(seq % (uint64_t)nwin);
            qvg_state &W = *win[wi];
            char *buf = static_cast<char *>(W.shards.bufs[0]);
            const uint64_t base_off = pdep_host(c, sg.outmask);
            if (overlap && prev) {
                // piece m overlaps old chunks pext(x, prev->outmask) for x in its range;
                // the last of them (bits varying inside the piece all 1) gates it
                const uint64_t lowvar = prev->outmask & (piece - 1);
                dep.resize(npieces);
                order.resize(npieces);
                for (uint64_t m = 0; m < npieces; ++m) {
                    dep[m] = pext_host(base_off + offhi[m] + lowvar, prev->outmask);
                    order[m] = m;
                }
                std::stable_sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) { return dep[a] < dep[b]; });
                uint64_t waited = ~0ull;
                for (uint64_t m : order) {
                    if (dep[m] != waited) {
                        cuda_check(cudaStreamWaitEvent(W.stream, done[0][dep[m]], 0), "cudaStreamWaitEvent");
                        waited = dep[m];
                    }
                    io.fetch_piece(W, buf, m, base_off + offhi[m], piece);
                }
            } else {
                io.fetch(W, wi, buf, base_off, offhi, piece);
            }
            chunk_ops(sg, ops, base_off, local);
            run_local(W, buf, local.data(), local.size());
            io.store(W, wi, buf, base_off, offhi, piece);
            if (overlap) cuda_check(cudaEventRecord(done[1][c], W.stream), "cudaEventRecord");
            host_bytes += 2 * (piece * npieces) * S;
        }
        if (overlap) {
            std::swap(done[0], done[1]);
            prev = &sg;
        } else {
            // the next segment regroups the qubits: every chunk must be home first
            for (int i = 0; i < nwin; ++i) cuda_check(cudaStreamSynchronize(win[i]->stream), "out-of-core sync");
            io.drain();
        }
    }
    for (int i = 0; i < nwin; ++i) cuda_check(cudaStreamSynchronize(win[i]->stream), "out-of-core sync");
    io.drain();
    if (stats_out) {
        *stats_out = qvg_stats{};
        for (int i = 0; i < nwin; ++i) {
            stats_out->passes += win[i]->stats.passes;
            stats_out->fused_passes += win[i]->stats.fused_passes;
            stats_out->kernel_launches += win[i]->stats.kernel_launches;
            stats_out->bytes_moved += win[i]->stats.bytes_moved;
        }
        stats_out->gates_applied = count;
        stats_out->exchanges = segs.size();      // round trips of the whole state through HBM
        stats_out->exchange_bytes = host_bytes;  // PCIe bytes, both directions
    }
}

int ooc_entry(uint32_t n, uint32_t precision, int device, uint32_t window_qubits, const qvg_gate *ops,
              uint64_t count, qvg_stats *stats_out, const std::function<std::unique_ptr<OocIo>(uint64_t)> &make_io) {
    qvg_state *win[3] = {nullptr, nullptr, nullptr};
    const int rc = guarded([&] {
        if (precision != QVG_C64 && precision != QVG_C128) throw Validation("precision must be 64 or 128");
        if (n < 1 || n > 48) throw Validation("n_qubits must be in [1, 48]");
        if (count && !ops) throw Validation("null op array");
        for (uint64_t i = 0; i < count; ++i) validate_op(ops[i], n, i);
        const uint32_t w = std::min(window_qubits, n);
        if (w < 4) throw Validation("window_qubits must be >= 4");
        // windows on their own streams: chunk k+1's copies and gates overlap
        // chunk k's. Three when they fit in 3/4 of the free HBM (chunk k+2's
        // H2D then need not wait for chunk k's D2H), else two.
        const uint64_t wbytes = ((uint64_t)(precision / 8)) << w;
        size_t free_b = 0, total_b = 0;
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
        const std::unique_ptr<OocIo> io = make_io(wbytes);
        // (caller I/O keeps two: its staging buffers are per window)
        const int nwin = (io->overlap_ok() && n - w >= 2 && 4 * 3 * wbytes <= 3 * (uint64_t)free_b) ? 3 : 2;
        for (int i = 0; i < nwin; ++i) {
            const int r = create_impl(w, precision, device, 0, 1, nullptr, false, &win[i]);
            if (r != QVG_OK) throw CudaFail(r, g_last_error);
        }
        ooc_run(*io, n, precision, w, ops, count, win, nwin, stats_out);
    });
    for (auto *ws : win)
        if (ws) qvg_destroy(ws);
    return rc;
}

}  // namespace

extern "C" {

int qvg_apply_host(void *host, uint32_t n, uint32_t precision, int device, uint32_t window_qubits,
                   const qvg_gate *ops, uint64_t count, qvg_stats *stats_out) {
    if (!host) {
        g_last_error = "null host state";
        return QVG_ERR_VALIDATION;
    }
    return ooc_entry(n, precision, device, window_qubits, ops, count, stats_out, [&](uint64_t) {
        return std::unique_ptr<OocIo>(new HostMemIo(host, precision / 8));
    });
}

int qvg_apply_stream(qvg_io_fn io, void *user, uint32_t n, uint32_t precision, int device, uint32_t window_qubits,
                     const qvg_gate *ops, uint64_t count, qvg_stats *stats_out) {
    if (!io) {
        g_last_error = "null I/O callback";
        return QVG_ERR_VALIDATION;
    }
    return ooc_entry(n, precision, device, window_qubits, ops, count, stats_out, [&](uint64_t window_bytes) {
        return std::unique_ptr<OocIo>(new CallbackIo(io, user, precision / 8, window_bytes));
    });
}

int qvg_device_memory(int device, uint64_t *free_bytes, uint64_t *total_bytes) {
    return guarded([&] {
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        size_t f = 0, t = 0;
        cuda_check(cudaMemGetInfo(&f, &t), "cudaMemGetInfo");
        if (free_bytes) *free_bytes = f;
        if (total_bytes) *total_bytes = t;
    });
}

int qvg_plan_passes(uint32_t n_qubits, uint32_t precision, int fuse, uint32_t tile_qubits, uint32_t carriers,
                    const qvg_gate *ops, uint64_t count, uint64_t *passes_out, uint64_t *fused_out,
                    uint64_t *bytes_out) {
    return guarded([&] {
        if (precision != QVG_C64 && precision != QVG_C128) throw Validation("precision must be 64 or 128");
        if (n_qubits < 1 || n_qubits > 40) throw Validation("n_qubits must be in [1, 40]");
        if (count && !ops) throw Validation("null op array");
        for (uint64_t i = 0; i < count; ++i) validate_op(ops[i], n_qubits, i);
        // the same options qvg_apply plans with on an unsharded state of this
        // precision and width (create_impl defaults + plan_options): 0 = default
        const TileShape shape = default_shape(precision);
        PlanOptions po;
        po.n = n_qubits;
        po.amp_bytes = precision == QVG_C128 ? 16 : 8;
        po.fuse = fuse != 0;
        po.tile_qubits = tile_qubits ? std::min<uint32_t>(tile_qubits, 12) : shape.tile_qubits;
        po.carriers = carriers ? carriers : shape.carriers;
        po.sub_bits = shape.sub_bits;
        small_state_shape(po, precision, n_qubits, tile_qubits != 0);
        const Plan plan = plan_ops(ops, count, po);  // as run_local (default reorder mode)
        uint64_t fused = 0, bytes = 0;
        for (const Pass &p : plan.passes) {
            fused += p.kind == PASS_TILE || p.kind == PASS_PERM;
            bytes += p.bytes;
        }
        if (passes_out) *passes_out = plan.passes.size();
        if (fused_out) *fused_out = fused;
        if (bytes_out) *bytes_out = bytes;
    });
}

int qvg_jit_info(uint64_t *compiled, uint64_t *failed, double *compile_ms, int *available) {
    return guarded([&] {
        const JitCounters c = jit_counters();
        if (compiled) *compiled = c.compiled;
        if (failed) *failed = c.failed;
        if (compile_ms) *compile_ms = c.compile_ms;
        if (available) *available = jit_available() ? 1 : 0;
    });
}

int qvg_jit_check(uint32_t n_qubits, uint32_t precision, const qvg_gate *ops, uint64_t count, uint64_t *passes_out,
                  uint64_t *compiled_out, char *err, uint64_t err_cap) {
    return guarded([&] {
        if (precision != QVG_C64 && precision != QVG_C128) throw Validation("precision must be 64 or 128");
        if (n_qubits < 1 || n_qubits > 40) throw Validation("n_qubits must be in [1, 40]");
        if (count && !ops) throw Validation("null op array");
        for (uint64_t i = 0; i < count; ++i) validate_op(ops[i], n_qubits, i);
        const TileShape shape = default_shape(precision);
        PlanOptions po;
        po.n = n_qubits;
        po.amp_bytes = precision == QVG_C128 ? 16 : 8;
        po.tile_qubits = shape.tile_qubits;
        po.carriers = shape.carriers;
        po.sub_bits = shape.sub_bits;
        small_state_shape(po, precision, n_qubits, false);
        const Plan plan = plan_ops(ops, count, po);
        uint64_t passes = 0, compiled = 0;
        std::string first;
        for (const Pass &p : plan.passes) {
            if (p.kind != PASS_TILE) continue;
            ++passes;
            const TileGeom &g = p.geom;
            const unsigned threads = 1u << (g.k - g.sub);
            const JitVariant jv{(int)po.amp_bytes, g.sub, false, threads <= 128 ? 128 : threads <= 256 ? 256 : 512,
                                kClsSets[class_set_index(g.cls_set)]};
            const std::string e = jit_compile(jit_source(g, plan.tile_ops.data() + p.op_begin, jv), nullptr);
            if (e.empty()) ++compiled;
            else if (first.empty()) first = e;
        }
        if (passes_out) *passes_out = passes;
        if (compiled_out) *compiled_out = compiled;
        if (err && err_cap) {
            const size_t n = std::min<size_t>(first.size(), err_cap - 1);
            std::memcpy(err, first.data(), n);
            err[n] = 0;
        }
    });
}

int qvg_set_step_hook(qvg_state *s, qvg_step_hook_fn fn, void *user) {
    return guarded([&] {
        check_state(s);
        s->hook = fn;
        s->hook_user = user;
    });
}

int qvg_exchange_plan(uint32_t n_qubits, uint32_t world, uint32_t rank, uint32_t precision, const qvg_shard_step *step,
                      uint64_t chunk_bytes, qvg_xchunk *out, uint64_t cap, uint64_t *count) {
    return guarded([&] {
        if (world < 2 || (world & (world - 1)) != 0) throw Validation("world size must be a power of two >= 2");
        if (rank >= world) throw Validation("rank out of range");
        if (precision != QVG_C64 && precision != QVG_C128) throw Validation("precision must be 64 or 128");
        if (!step) throw Validation("null step");
        uint32_t g = 0;
        while ((1u << g) < world) ++g;
        if (n_qubits < g + 2 || n_qubits > 40) throw Validation("too few qubits for this many shards");
        if (step->type == STEP_EXCHANGE && (step->gpos >= n_qubits))
            throw Validation("exchange step: gpos out of range");
        if (step->type == STEP_MULTI_EXCHANGE && (step->gpos >> g) != 0)
            throw Validation("multi-exchange mask has bits beyond the rank bits");
        if (chunk_bytes == 0 || chunk_bytes % 16) throw Validation("chunk_bytes must be a positive multiple of 16");
        std::vector<XChunk> plan;
        try {
            plan = exchange_chunks(n_qubits - g, precision == QVG_C128 ? 16 : 8, chunk_bytes, rank, *step);
        } catch (const std::invalid_argument &e) {
            throw Validation(e.what());
        }
        if (count) *count = plan.size();
        static_assert(sizeof(XChunk) == sizeof(qvg_xchunk), "qvg_xchunk layout");
        if (out) std::memcpy(out, plan.data(), std::min<uint64_t>(cap, plan.size()) * sizeof(XChunk));
    });
}

int qvg_shard_schedule(uint32_t n_qubits, uint32_t world, const qvg_gate *ops, uint64_t count, int canonicalize,
                       qvg_shard_step *steps, uint64_t cap, uint64_t *nsteps) {
    return guarded([&] {
        if (world == 0 || (world & (world - 1)) != 0) throw Validation("world size must be a power of two");
        uint32_t g = 0;
        while ((1u << g) < world) ++g;
        if (n_qubits < g + 2 || n_qubits > 40) throw Validation("too few qubits for this many shards");
        if (count && !ops) throw Validation("null op array");
        for (uint64_t i = 0; i < count; ++i) validate_op(ops[i], n_qubits, i);
        const uint32_t L = n_qubits - g;
        QubitMap map;
        map.reset(n_qubits);
        std::vector<ShardStep> out;
        // flags: bit 0 canonicalize; bits 8..11 the most global qubits one
        // exchange may swap (0 or 1: pairwise exchanges only)
        const uint32_t kmax = std::max<uint32_t>(1, ((uint32_t)canonicalize >> 8) & 0xf);
        schedule_ops(n_qubits, L, ops, count, map, out, kmax);
        if (canonicalize & 1) schedule_canonicalize(n_qubits, L, map, out, kmax);
        if (nsteps) *nsteps = out.size();
        if (steps) std::memcpy(steps, out.data(), std::min<uint64_t>(cap, out.size()) * sizeof(ShardStep));
    });
}

}  // extern "C"
