/*
 * qvg.h — C-ABI of the B200-native gate-application engine (libqvg.so).
 *
 * This is the drop-in boundary for the QVecOpt reference's hot path
 * (arXiv 2508.15545, /root/reference/proj). The reference has no FFI; its
 * boundary is the C++ API listed beside each entry point below. The C++ host
 * layer (paper_2508_15545_b200/csrc/host/) adds `Strategy::gpu` to the
 * reference's `apply_circuit` dispatch and calls these functions; the pybind11
 * module exposes the same names the reference's `qvsim._core` does.
 *
 * Conventions
 *   - Plain C types only: pointers, sizes, status codes. No torch, no C++.
 *   - Qubit 0 is the least-significant bit of the amplitude index
 *     (reference SPEC.md:96, types.hpp:19-26).
 *   - Amplitudes are interleaved (re, im) pairs, little-endian, in the state's
 *     precision: complex128 = 2 x double (16 B, reference types.hpp:13-16),
 *     complex64 = 2 x float (8 B, not in the reference; added for config 2).
 *   - Every call returns QVG_OK or a status that maps 1:1 onto the reference's
 *     error tree (reference include/qvsim/error.hpp:10-50); the message is in
 *     qvg_last_error() (thread-local).
 *   - One qvg_state is owned by one host thread (the reference's CacheWindow
 *     single-owner rule, cache.hpp:44-47). Work is stream-ordered on the
 *     state's CUDA stream; qvg_sync() waits for it.
 */
#ifndef QVG_H
#define QVG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QVG_ABI_VERSION 3  /* 3: qvg_exchange_plan, qvg_set_step_hook, QVG_OPT_XCHG_CHUNK, per-segment
                              sharded timing (kernel_ms / exchange_ms); 2: qvg_stats.fused_exchanges,
                              multi-exchange steps, options 10-13 */

/* Status codes -> reference exception types (error.hpp:10-50). */
enum qvg_status {
    QVG_OK = 0,
    QVG_ERR_VALIDATION = 1, /* qvsim::ValidationError: bad qubit, size, op */
    QVG_ERR_CAPACITY = 2,   /* qvsim::CapacityError: device memory too small */
    QVG_ERR_IO = 3,         /* qvsim::IoError: CUDA / NCCL runtime failure */
    QVG_ERR_FORMAT = 4,     /* qvsim::FormatError: bad state-file header */
    QVG_ERR_NO_DEVICE = 5   /* qvsim::IoError: no CUDA device / bad build */
};

/* Op kinds (reference types.hpp:41 OpKind). */
enum qvg_op_kind { QVG_OP_SINGLE = 0, QVG_OP_CONTROLLED = 1 };

/* Flattened qvsim::GateOp (reference types.hpp:43-52). The name/params text
 * form stays on the host; the device only needs the matrix and the qubits.
 * u[] is the row-major 2x2 matrix as 8 reals in the reference's "u" order
 * (gates.hpp:26-29): re00 im00 re01 im01 re10 im10 re11 im11. */
typedef struct qvg_gate {
    uint32_t kind;    /* qvg_op_kind */
    uint32_t target;  /* GateOp::target */
    int32_t control;  /* GateOp::control, -1 when absent */
    uint32_t flags;   /* reserved, must be 0 */
    double u[8];
} qvg_gate;

/* Precision tags for qvg_create. */
enum qvg_precision { QVG_C64 = 64, QVG_C128 = 128 };

/* Option keys for qvg_set_option. */
enum qvg_option {
    QVG_OPT_FUSE = 1,        /* 1: fused low/strided tile passes (default), 0: one pass per gate */
    QVG_OPT_TILE_QUBITS = 2, /* qubits per fused tile, 5..12 (default 11; complex64 12) */
    QVG_OPT_CARRIERS = 3,    /* lowest qubits every tile keeps contiguous (default 3) */
    QVG_OPT_LOW_KERNEL = 4,  /* 1: warp-shuffle kernel for targets < 5, 0: k_pairs (default, measured faster) */
    QVG_OPT_MIN_RUN = 5,     /* bytes: a control/phase bit whose 1-runs are shorter is selected
                                inside a dense pass instead of enumerated (default 32) */
    QVG_OPT_PRED_STORE = 6,  /* 1: skip stores of unselected amplitudes; 0: write them back (default) */
    QVG_OPT_SUB_BITS = 7,    /* fused tile: 2^b register amplitudes per thread, b = 3 or 4 (default 4);
                                complex64 also 5 (its default) */
    QVG_OPT_FMA = 8,         /* 1: fused-tile complex128 arithmetic with DFMA (faster, within 1e-15
                                relative but NOT bit-identical to the reference); 0: exact (default) */
    QVG_OPT_TIMING = 9,      /* 1: CUDA events around each qvg_apply (sharded: around every local-pass
                                batch and exchange); qvg_stats.kernel_ms / exchange_ms sum them */
    QVG_OPT_EXCHANGE = 10,   /* sharded states: 0 copy exchange (NCCL send/recv; virtual: swap kernel),
                                1 peer-memory exchange kernel, 2 peer exchange fused with the gate that
                                triggered it, -1 auto (default: 2 for NCCL ranks whose peers map, else 1) */
    QVG_OPT_PREFETCH = 11,   /* fused tile: 1 = load the next tile's first-group amplitudes into
                                registers during the current tile (8-amplitude subcubes only) */
    QVG_OPT_BATCH_EXCHANGE = 12, /* sharded: most global qubits one exchange swaps, 1..4 (default 4; 1 =
                                    pairwise exchanges only) */
    QVG_OPT_STAGE = 13,      /* fused tile: a first/last register group holding tile bits 0..b-1 moves
                                its HBM data through shared memory, coalesced (default b = 3; 0 never) */
    QVG_OPT_GRAPH = 14,      /* unsharded states: replay an op list as a captured CUDA graph (no per-pass host
                                planning / launch cost): 2 = auto (default; lists of >= 8 ops, from their second
                                apply on this state), 1 = every list, 0 = never */
    QVG_OPT_REORDER = 15,    /* fusion may move an op ahead of ops on disjoint qubits (fewer passes):
                                2 = only moves that keep every bit (an X/CX permutation or a Z/CZ sign
                                flip on either side; default), 1 = any such move (mathematically equal,
                                NOT bit-identical to the reference), 0 = circuit order */
    QVG_OPT_CLASSES = 16,    /* fused tile: 1 = structured-matrix op bodies (real, X, entries +-1/2, Z),
                                same values with fewer FP64 instructions (default); 0 = general bodies */
    QVG_OPT_XCHG_CHUNK = 17, /* sharded: copy-transport chunk bytes (multiple of 16; 0 = default 256 MiB,
                                capped by the NCCL scratch); tests use small chunks to split runs */
    QVG_OPT_JIT = 19,        /* fused tiles: run a pass as a kernel specialised to its op list (NVRTC,
                                cached per pass structure, compiled in parallel before an apply's first
                                launch; bit-identical to k_tile): 1 (= 2) the passes of >= 2^24-amplitude
                                states jit_pays picks (complex64; complex128 passes of X / real / diagonal
                                ops), 3 = every pass, 0 = never (default: no net gain measured,
                                profiles/r02_jit_ab.json) */
    QVG_OPT_PERM = 20,       /* 1: a fused run of only X / CX / Z / CZ ops runs as one shared-memory scatter
                                (k_tile_perm, bit-identical to k_tile), 0: through k_tile (default: the
                                scatter measured equal, profiles/r02_perm_ab.json) */
    QVG_OPT_TILE_ORDER = 21, /* fused tiles: 0 = CTA b runs tiles b, b + grid, ... (default); 1 = a contiguous
                                chunk of tiles per CTA (successive tiles are DRAM neighbours) */
    QVG_OPT_TILE_GRID = 22,  /* fused tiles: 0 = one persistent wave of CTAs loops over the tiles, 1 = one
                                CTA per tile (up to 16 tiles per CTA while several waves of CTAs remain), -1 = auto (default: 1) */
    QVG_OPT_PIPE = 18        /* fused tiles, data movement: 0 = k_tile (per-thread loads); 2 or 3 =
                                warp-specialised bulk-copy ring with that many stages (k_tile_pipe) and 4 =
                                tensor-map TMA (both measured slower, profiles/r02_pipe_ab.json); 5 =
                                k_tile_ahead (the next tile's cp.async load runs under the last register
                                group, same occupancy) for every pass, 6 = for passes light in FP64 work;
                                -1 = auto (default: 6 for complex128, 0 for complex64) */
};

/* Counters (the reference's Metrics, metrics.hpp:14-30, plus the GPU pass
 * accounting of SURVEY §5). Cumulative over the state's lifetime. */
typedef struct qvg_stats {
    uint64_t gates_applied;  /* Metrics::gates_applied */
    uint64_t passes;         /* HBM passes launched (Metrics::traversals analog) */
    uint64_t fused_passes;   /* of which fused tile passes */
    uint64_t kernel_launches;
    uint64_t bytes_moved;    /* algorithmic HBM bytes, read + write */
    uint64_t exchange_bytes; /* bytes sent over NVLink (sharded states) */
    uint64_t exchanges;      /* pairwise half-shard exchanges */
    double kernel_ms;        /* device time of gate passes (QVG_OPT_TIMING states only) */
    double exchange_ms;      /* device time of exchanges (QVG_OPT_TIMING, sharded states) */
    uint64_t fused_exchanges; /* exchanges that also applied the gate that caused them (k_xchg) */
    uint64_t graph_replays;   /* applies that ran as a captured CUDA graph (QVG_OPT_GRAPH) */
    uint64_t jit_passes;      /* fused passes that ran as a JIT-specialised kernel (QVG_OPT_JIT) */
} qvg_stats;

typedef struct qvg_state qvg_state;

/* ---- lifecycle ------------------------------------------------------------
 * Replaces BlockStore::create (reference store.hpp:55-57, store.cpp:181-214):
 * allocates 2^n amplitudes in HBM and initialises |0...0> (amp[0] = 1). */
int qvg_create(uint32_t n_qubits, uint32_t precision, int device, qvg_state **out);

/* Sharded state over `world` ranks, one process per GPU. Rank r
 * owns global indices [r*2^L, (r+1)*2^L), L = n - log2(world) (reference
 * parallel.cpp:13-37, Eq. 9). nccl_id is the 128-byte ncclUniqueId made by
 * qvg_nccl_unique_id on rank 0 and broadcast by the caller. */
int qvg_create_sharded(uint32_t n_qubits, uint32_t precision, int device,
                       uint32_t rank, uint32_t world, const void *nccl_id,
                       qvg_state **out);
int qvg_nccl_unique_id(void *out128);
int qvg_destroy(qvg_state *s);

/* Shape queries. */
int qvg_info(const qvg_state *s, uint32_t *n_qubits, uint32_t *precision,
             uint32_t *rank, uint32_t *world);

/* Options (qvg_option). */
int qvg_set_option(qvg_state *s, int key, int64_t value);

/* ---- state init / transfer -------------------------------------------------
 * |index> basis state (BlockStore::create gives index 0). Global index. */
int qvg_init_basis(qvg_state *s, uint64_t index);
/* Host -> device copy of amplitudes [offset, offset+count) in the state's
 * precision (write_full_state, reference engine.cpp:496-509). For sharded
 * states the range is global; each rank copies the part it owns. */
int qvg_load(qvg_state *s, const void *host, uint64_t offset, uint64_t count);
/* Device -> host (read_full_state, reference engine.cpp:483-494). */
int qvg_read(qvg_state *s, void *host, uint64_t offset, uint64_t count);
/* Stream-ordered variants: enqueue the copy on the state's stream and return;
 * `host` must stay valid until qvg_sync and should be pinned for full PCIe
 * bandwidth. Two states on their own streams then overlap one state's copies
 * with the other's gates (PCIe is full duplex). */
int qvg_load_async(qvg_state *s, const void *host, uint64_t offset, uint64_t count);
int qvg_read_async(qvg_state *s, void *host, uint64_t offset, uint64_t count);

/* Out-of-core apply (the paper's sliding window over a block
 * store, lifted to host memory -> HBM): the state is 2^n amplitudes in HOST
 * memory (page-locked for full PCIe bandwidth), the device holds two windows
 * of 2^window_qubits amplitudes. Each segment of the circuit whose
 * non-diagonal targets fit one window streams the whole state host -> HBM ->
 * host once, chunk by chunk, with the fused planner inside each chunk. Results
 * are bit-identical to qvg_apply on a device-resident state. stats_out (may
 * be NULL): passes/bytes of the device work; exchanges = segments,
 * exchange_bytes = PCIe bytes. */
int qvg_apply_host(void *host_state, uint32_t n_qubits, uint32_t precision, int device,
                   uint32_t window_qubits, const qvg_gate *ops, uint64_t count, qvg_stats *stats_out);

/* Out-of-core apply with caller I/O: the state lives wherever `io` reads and
 * writes it (e.g. a QVSV file via pread/pwrite, the paper's disk tier).
 * io(user, offset, count, buf, write) moves `count` amplitudes at amplitude
 * offset `offset` between the store and `buf` (write = 0: store -> buf) and
 * returns 0 on success. Same segment planning and results as qvg_apply_host;
 * two pinned staging buffers of 2^window_qubits amplitudes let the file I/O of
 * one chunk overlap the device work on another. */
typedef int (*qvg_io_fn)(void *user, uint64_t offset, uint64_t count, void *buf, int write);
int qvg_apply_stream(qvg_io_fn io, void *user, uint32_t n_qubits, uint32_t precision, int device,
                     uint32_t window_qubits, const qvg_gate *ops, uint64_t count, qvg_stats *stats_out);
/* Free / total device memory (cudaMemGetInfo), to size windows or pick a path. */
int qvg_device_memory(int device, uint64_t *free_bytes, uint64_t *total_bytes);

/* Page-locked host memory for the async copies (cudaHostAlloc / cudaFreeHost). */
int qvg_host_alloc(uint64_t bytes, void **out);
int qvg_host_free(void *ptr);

/* ---- the hot path ------------------------------------------------------------
 * Apply `count` ops in order (reference apply_circuit for a whole circuit,
 * engine.cpp:86-157; apply_gate_streamed for count == 1, kernel.cpp:132-146).
 * Validates every op first (reference kernel.cpp:134-140, circuit.cpp:31-52)
 * and enqueues nothing on error. Stream-ordered: returns once the work is
 * enqueued; qvg_sync() waits. */
int qvg_apply(qvg_state *s, const qvg_gate *ops, uint64_t count);
int qvg_sync(qvg_state *s);

/* ---- readout ------------------------------------------------------------------
 * |a_i|^2 = re*re + im*im (std::norm, reference engine.cpp:518) for
 * i in [offset, offset+count), written as doubles. Synchronous. */
int qvg_probabilities(qvg_state *s, double *out, uint64_t offset, uint64_t count);
/* sqrt(sum |a_i|^2) (BlockStore::norm, reference store.cpp:301-316). */
int qvg_norm(qvg_state *s, double *out);
/* The k largest |a_i|^2, descending, ties by ascending index
 * (top_amplitudes, reference engine.cpp:511-544). amps_out gets 2*k reals. */
int qvg_top_amplitudes(qvg_state *s, uint32_t k, uint64_t *index_out,
                       double *amps_out);

/* <a|b> = sum_i conj(a_i) b_i for two states of the same shape (
 * fidelity = |<a|b>|^2, the north_star parity measure). */
int qvg_inner_product(qvg_state *a, qvg_state *b, double *re, double *im);
/* max_i |a_i - b_i| (max_deviation, reference dense.cpp:174-183). */
int qvg_max_deviation(qvg_state *a, qvg_state *b, double *out);

/* Chunk checksums of the state in canonical order: for every chunk of
 * `chunk_amps` amplitudes (a power of two >= 4096), two 64-bit words of
 * order-independent sums of mixed amplitude bit patterns (qvg_readout.cuh
 * k_checksum; numpy restatement in tests/conftest.py). out[2c], out[2c+1]
 * for chunk c; `cap` counts chunks; *count = 2^n / chunk_amps (call with
 * out = NULL to size). A size-independent parity property: equal states
 * have equal words, and any bit change shows with probability ~1 - 2^-128. */
int qvg_checksums(qvg_state *s, uint64_t chunk_amps, uint64_t *out, uint64_t cap, uint64_t *count);

/* ---- instrumentation --------------------------------------------------------- */
int qvg_stats_get(const qvg_state *s, qvg_stats *out);
int qvg_stats_reset(qvg_state *s);
/* The cudaStream_t the state's work runs on (for CUDA-event timing). */
int qvg_stream(const qvg_state *s, void **stream_out);
/* Device pointer and byte size of this rank's amplitude shard. */
int qvg_device_buffer(const qvg_state *s, void **ptr_out, uint64_t *bytes_out);
/* JIT-specialised tile passes (QVG_OPT_JIT, paper_2508_15545_b200/csrc/qvg_jit.hpp):
 * process-wide counters (kernels compiled / failed, summed per-kernel compile
 * ms); available = NVRTC and the driver entry points loaded. */
int qvg_jit_info(uint64_t *compiled, uint64_t *failed, double *compile_ms, int *available);
/* Host-only check of the JIT source path (no GPU needed): plans the ops as
 * qvg_apply would on an unsharded state of this width/precision (defaults,
 * fusion on), generates every fused pass's specialised source and compiles
 * it with NVRTC for sm_100a. *passes_out = fused passes, *compiled_out = those
 * that compiled; the first error log goes to err (NUL-terminated, cap bytes). */
int qvg_jit_check(uint32_t n_qubits, uint32_t precision, const qvg_gate *ops, uint64_t count,
                  uint64_t *passes_out, uint64_t *compiled_out, char *err, uint64_t err_cap);
/* Number of gate passes qvg_apply would launch for these ops (planner only,
 * no device work; usable without a GPU). */
int qvg_plan_passes(uint32_t n_qubits, uint32_t precision, int fuse,
                    uint32_t tile_qubits, uint32_t carriers, const qvg_gate *ops,
                    uint64_t count, uint64_t *passes_out, uint64_t *fused_out,
                    uint64_t *bytes_out);
/* Schedule of a state sharded over `world` = 2^g ranks, as run
 * by qvg_apply on a sharded state; host-only, usable without a GPU. */
enum qvg_step_type { QVG_STEP_LOCAL = 0, QVG_STEP_EXCHANGE = 1, QVG_STEP_LOCAL_SWAP = 2, QVG_STEP_MULTI_EXCHANGE = 3 };
typedef struct qvg_shard_step {
    uint32_t type;       /* qvg_step_type */
    uint32_t rank_mask;  /* LOCAL: runs on ranks with (rank & rank_mask) == rank_value */
    uint32_t rank_value;
    uint32_t gpos;       /* EXCHANGE: global physical qubit (>= L); MULTI_EXCHANGE: the swapped global
                            qubits as a rank-bit mask (bit j = physical qubit L + j) */
    uint32_t lpos;       /* EXCHANGE: local qubit swapped with gpos; LOCAL_SWAP: first local qubit;
                            MULTI_EXCHANGE: the local qubits, 8 bits each, in the mask's bit order */
    uint32_t lpos2;      /* LOCAL_SWAP: second local qubit; MULTI_EXCHANGE: k, the number of pairs */
    qvg_gate op;         /* LOCAL: op on physical local qubits */
} qvg_shard_step;
/* Steps for ops[0..count) from the identity qubit map. `canonicalize` is a
 * flag word: bit 0 appends the steps that restore the canonical order; bits
 * 8..11 give the most global qubits one exchange may swap (0/1: pairwise). Writes at most `cap`
 * steps and the total count to *nsteps (call with cap = 0 to size). */
int qvg_shard_schedule(uint32_t n_qubits, uint32_t world, const qvg_gate *ops, uint64_t count,
                       int canonicalize, qvg_shard_step *steps, uint64_t cap, uint64_t *nsteps);
/* The copy transport's chunk plan for one exchange step on one rank
 * (qvg_schedule.hpp exchange_chunks), in issue order: chunk i is one grouped
 * send/recv with `partner` of the `bytes` at `offset_bytes` of this rank's
 * shard, received into the same place; chunk i of a rank and of its partner
 * carry each other's data. The plan the NCCL and virtual-shard copy
 * transports execute; host-only (tests drive it over gloo). Writes at most
 * `cap` entries and the total to *count. */
typedef struct qvg_xchunk {
    uint32_t round;   /* 1-based round (multi-exchange: 1 .. 2^k - 1) */
    uint32_t partner;
    uint64_t offset_bytes;
    uint64_t bytes;
} qvg_xchunk;
int qvg_exchange_plan(uint32_t n_qubits, uint32_t world, uint32_t rank, uint32_t precision,
                      const qvg_shard_step *step, uint64_t chunk_bytes, qvg_xchunk *out,
                      uint64_t cap, uint64_t *count);
/* Test instrumentation around every executed segment of a sharded apply (a
 * batch of local passes or one exchange; the reference's ExecHooks,
 * parallel.hpp:40-45): fn(user, rank, segment, step_type, phase) with phase 0
 * before the segment is enqueued and 1 after its device work completed (the
 * state's stream is synchronised while a hook is installed). A nonzero
 * return is an injected fault: qvg_apply fails with QVG_ERR_IO and no later
 * segment runs. NULL removes the hook. */
typedef int (*qvg_step_hook_fn)(void *user, uint32_t rank, uint64_t segment, uint32_t step_type, uint32_t phase);
int qvg_set_step_hook(qvg_state *s, qvg_step_hook_fn fn, void *user);
/* Thread-local message of the last failing call ("" when none). */
const char *qvg_last_error(void);
int qvg_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* QVG_H */
