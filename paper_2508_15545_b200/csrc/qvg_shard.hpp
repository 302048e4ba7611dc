// qvg_shard.hpp — state sharding over G = 2^g GPUs, executing
// the host schedule of qvg_schedule.hpp.
//
// Three transports behind one executor:
//   * peer memory (one process per GPU, the deployment mode on an NVSwitch
//     box): the shards are mapped into every rank with CUDA IPC, and a
//     global-target gate runs as ONE kernel (k_xchg) that exchanges the
//     half-shards and applies the gate in the same pass. Each rank of a pair
//     streams half of the pairs, half its bytes over NVLink. Stream-ordered
//     NCCL barriers go before and after the kernel;
//   * NCCL copy (when peers cannot be mapped): pairwise half-shard exchange
//     with ncclSend/ncclRecv over NVLink, chunked through a scratch buffer;
//   * virtual shards (all G shards on this device, one process): the same
//     schedule and the same k_xchg kernel, with the "peer" pointer being
//     another buffer on this device and one launch per rank role. This is how
//     the sharded path, including the fused exchange, is tested bit-for-bit on
//     a single GPU (the profiling guide forbids emulating ranks as processes
//     that wait on each other).
// The reference's only "nodes" are threads over one shared file
// (reference parallel.cpp:55-143); it never exchanges data.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <queue>
#include <string>
#include <vector>

#include "qvg.h"
#include "qvg_kernels.cuh"
#include "qvg_plan.hpp"
#include "qvg_readout.cuh"
#include "qvg_schedule.hpp"

struct qvg_state;

namespace qvg {

// Hooks implemented in qvg_engine.cu.
void shard_run_local(qvg_state &s, void *psi, const qvg_gate *ops, uint64_t count);
cudaStream_t shard_stream(qvg_state &s);
uint32_t shard_amp_bytes(const qvg_state &s);
qvg_stats &shard_stats(qvg_state &s);
int shard_exchange_mode(const qvg_state &s);  // QVG_OPT_EXCHANGE value (-1 = auto)
uint32_t shard_batch_max(const qvg_state &s);  // QVG_OPT_BATCH_EXCHANGE: most global qubits per exchange
void cuda_throw(cudaError_t e, const char *what);
// QVG_OPT_TIMING on a sharded state: CUDA events around every executed
// segment (a batch of local passes, or an exchange), folded into
// qvg_stats.kernel_ms (kind 0) and exchange_ms (kind 1) by qvg_stats_get.
bool shard_timing(const qvg_state &s);
void shard_time_push(qvg_state &s, cudaEvent_t a, cudaEvent_t b, int kind);
// qvg_set_step_hook: test instrumentation around every executed segment
// (the reference's ExecHooks, parallel.hpp:40-45). Returns the hook's value.
bool shard_has_hook(const qvg_state &s);
int shard_step_hook(qvg_state &s, uint32_t rank, uint64_t segment, uint32_t type, uint32_t phase);

inline void nccl_check(ncclResult_t r, const char *what) {
    if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + ncclGetErrorString(r));
}

struct ShardSet {
    uint32_t n = 0, L = 0, rank = 0, world = 1;
    bool is_virtual = false;
    std::vector<void *> bufs;    // local shard buffers (1, or `world` when virtual)
    std::vector<uint32_t> ranks; // rank of each local buffer
    QubitMap map;
    ncclComm_t comm = nullptr;
    void *scratch = nullptr;
    uint64_t scratch_bytes = 0;
    uint64_t chunk_bytes = 0;
    uint64_t chunk_override = 0;  // QVG_OPT_XCHG_CHUNK: copy-transport chunk bytes (tests)
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t received[2] = {nullptr, nullptr}, copied[2] = {nullptr, nullptr};
    double *d_scalar = nullptr;
    std::vector<void *> peer;  // NCCL mode: every rank's shard, mapped here via CUDA IPC (own = bufs[0])
    bool peer_ok = false;

    void init(qvg_state &s, uint32_t n_, uint32_t L_, uint32_t rank_, uint32_t world_, const void *nccl_id,
              bool virt) {
        n = n_;
        L = L_;
        rank = rank_;
        world = world_;
        is_virtual = virt && world > 1;
        map.reset(n);
        const uint64_t bytes = (uint64_t)shard_amp_bytes(s) << L;
        const uint32_t nbuf = is_virtual ? world : 1;
        for (uint32_t b = 0; b < nbuf; ++b) {
            void *p = nullptr;
            cuda_throw(cudaMalloc(&p, bytes), "cudaMalloc(state shard)");
            bufs.push_back(p);
            ranks.push_back(is_virtual ? b : rank);
        }
        if (world > 1 && !is_virtual) {
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof(id));
            nccl_check(ncclCommInitRank(&comm, (int)world, id, (int)rank), "ncclCommInitRank");
            chunk_bytes = std::min<uint64_t>(bytes / 2, 256ull << 20);
            scratch_bytes = 2 * chunk_bytes;  // double-buffered
            cuda_throw(cudaMalloc(&scratch, scratch_bytes), "cudaMalloc(exchange scratch)");
            cuda_throw(cudaMalloc(&d_scalar, 64), "cudaMalloc(scalar)");
            cuda_throw(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking), "cudaStreamCreate(copy)");
            for (int b = 0; b < 2; ++b) {
                cuda_throw(cudaEventCreateWithFlags(&received[b], cudaEventDisableTiming), "cudaEventCreate");
                cuda_throw(cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming), "cudaEventCreate");
            }
            open_peers();
        }
    }

    // Map every rank's shard into this process (cudaIpcGetMemHandle, an
    // ncclAllGather of the handles, cudaIpcOpenMemHandle). All ranks agree on
    // the outcome (allreduce of a failure count); on failure the NCCL copy
    // transport is used.
    void open_peers() {
        cudaIpcMemHandle_t mine{};
        double fail = cudaIpcGetMemHandle(&mine, bufs[0]) == cudaSuccess ? 0.0 : 1.0;
        (void)cudaGetLastError();
        std::vector<cudaIpcMemHandle_t> all(world);
        char *d = nullptr;
        cuda_throw(cudaMalloc(&d, sizeof(cudaIpcMemHandle_t) * (world + 1)), "cudaMalloc(ipc handles)");
        cuda_throw(cudaMemcpy(d, &mine, sizeof(mine), cudaMemcpyHostToDevice), "H2D ipc handle");
        nccl_check(ncclAllGather(d, d + sizeof(mine), sizeof(mine), ncclChar, comm, nullptr), "ncclAllGather(ipc)");
        cuda_throw(cudaMemcpy(all.data(), d + sizeof(mine), sizeof(mine) * world, cudaMemcpyDeviceToHost),
                   "D2H ipc handles");
        peer.assign(world, nullptr);
        peer[rank] = bufs[0];
        for (uint32_t r = 0; r < world && fail == 0.0; ++r) {
            if (r == rank) continue;
            if (cudaIpcOpenMemHandle(&peer[r], all[r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                (void)cudaGetLastError();
                peer[r] = nullptr;
                fail = 1.0;
            }
        }
        cuda_throw(cudaMemcpy(d, &fail, sizeof(fail), cudaMemcpyHostToDevice), "H2D flag");
        nccl_check(ncclAllReduce(d, d, 1, ncclDouble, ncclSum, comm, nullptr), "ncclAllReduce(ipc ok)");
        cuda_throw(cudaMemcpy(&fail, d, sizeof(fail), cudaMemcpyDeviceToHost), "D2H flag");
        cudaFree(d);
        peer_ok = fail == 0.0;
        if (!peer_ok) close_peers();
    }

    void close_peers() {
        for (uint32_t r = 0; r < peer.size(); ++r)
            if (peer[r] && r != rank) cudaIpcCloseMemHandle(peer[r]);
        peer.clear();
        peer_ok = false;
    }

    void release() {
        close_peers();
        for (void *p : bufs) cudaFree(p);
        bufs.clear();
        ranks.clear();
        if (scratch) cudaFree(scratch);
        scratch = nullptr;
        scratch_bytes = 0;
        if (copy_stream) cudaStreamDestroy(copy_stream);
        copy_stream = nullptr;
        for (int b = 0; b < 2; ++b) {
            if (received[b]) cudaEventDestroy(received[b]);
            if (copied[b]) cudaEventDestroy(copied[b]);
            received[b] = copied[b] = nullptr;
        }
        if (d_scalar) cudaFree(d_scalar);
        d_scalar = nullptr;
        if (comm) ncclCommDestroy(comm);
        comm = nullptr;
    }

    // Chunk size of the copy transport: the NCCL scratch halves; virtual
    // shards use the same 256 MiB cap (or a test override).
    uint64_t copy_chunk_bytes(uint32_t S) const {
        if (chunk_override) return chunk_bytes ? std::min(chunk_override, chunk_bytes) : chunk_override;
        if (chunk_bytes) return chunk_bytes;
        return std::min<uint64_t>(((uint64_t)S << L) / 2, 256ull << 20);
    }
    void ensure_scratch(uint64_t bytes) {
        if (scratch_bytes >= bytes) return;
        if (scratch) cudaFree(scratch);
        scratch = nullptr;
        scratch_bytes = 0;
        cuda_throw(cudaMalloc(&scratch, bytes), "cudaMalloc(exchange scratch)");
        scratch_bytes = bytes;
    }

    std::vector<void *> local_buffers() const { return bufs; }
    std::vector<uint32_t> local_ranks() const { return ranks; }
};

inline void shard_nccl_unique_id(void *out) {
    ncclUniqueId id;
    nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
}

inline void shard_init_basis(qvg_state &s, ShardSet &set, uint64_t index) {
    cudaStream_t st = shard_stream(s);
    const uint32_t S = shard_amp_bytes(s);
    const uint64_t bytes = (uint64_t)S << set.L;
    set.map.reset(set.n);
    for (size_t b = 0; b < set.bufs.size(); ++b) {
        cuda_throw(cudaMemsetAsync(set.bufs[b], 0, bytes, st), "cudaMemsetAsync(state)");
        if ((index >> set.L) == set.ranks[b]) {
            const uint64_t local = index & ((1ull << set.L) - 1);
            static const double one_d[2] = {1.0, 0.0};
            static const float one_f[2] = {1.0f, 0.0f};
            cuda_throw(cudaMemcpyAsync(static_cast<char *>(set.bufs[b]) + local * S, S == 16 ? (const void *)one_d
                                                                                             : (const void *)one_f,
                                       S, cudaMemcpyHostToDevice, st),
                       "cudaMemcpyAsync(basis amplitude)");
        }
    }
}

template <class R>
inline void launch_swap_bits(cudaStream_t st, void *psi, uint32_t L, uint32_t a, uint32_t b) {
    using T = typename Cplx<R>::T;
    if (a > b) std::swap(a, b);
    const uint64_t count = 1ull << (L - 2);
    if (count >= 1024)
        k_swap_bits<R, 4><<<(unsigned)(count / 1024), 256, 0, st>>>(static_cast<T *>(psi), (int)a, (int)b);
    else {
        const unsigned bs = (unsigned)std::min<uint64_t>(count, 256);
        k_swap_bits<R, 1><<<(unsigned)(count / bs), bs, 0, st>>>(static_cast<T *>(psi), (int)a, (int)b);
    }
}

inline void run_local_swap(qvg_state &s, ShardSet &set, uint32_t a, uint32_t b) {
    cudaStream_t st = shard_stream(s);
    for (void *psi : set.bufs) {
        if (shard_amp_bytes(s) == 16) launch_swap_bits<double>(st, psi, set.L, a, b);
        else launch_swap_bits<float>(st, psi, set.L, a, b);
    }
    cuda_throw(cudaGetLastError(), "swap_bits launch");
    shard_stats(s).passes += set.bufs.size();
    shard_stats(s).kernel_launches += set.bufs.size();
    shard_stats(s).bytes_moved += set.bufs.size() * ((uint64_t)shard_amp_bytes(s) << set.L);
}

template <class R>
inline void launch_xchg(cudaStream_t st, void *a, void *b, uint32_t lpos, uint64_t t0, uint64_t nt, int cbit,
                        int mode, const double *u, int fence) {
    using T = typename Cplx<R>::T;
    Mat<R> m;
    for (int i = 0; i < 8; ++i) m.u[i] = u ? (R)u[i] : R(0);
    T *pa = static_cast<T *>(a), *pb = static_cast<T *>(b);
    if (nt >= 1024) {
        k_xchg<R, 4><<<(unsigned)(nt / 1024), 256, 0, st>>>(pa, pb, (int)lpos, t0, cbit, mode, fence, m);
    } else {
        const unsigned bs = (unsigned)std::min<uint64_t>(nt, 256);
        k_xchg<R, 1><<<(unsigned)(nt / bs), bs, 0, st>>>(pa, pb, (int)lpos, t0, cbit, mode, fence, m);
    }
}

// Stream-ordered barrier over all ranks: a one-element allreduce completes on
// a rank only after every rank's earlier work on its state stream is done.
inline void stream_barrier(ShardSet &set, cudaStream_t st) {
    nccl_check(ncclAllReduce(set.d_scalar, set.d_scalar, 1, ncclDouble, ncclSum, set.comm, st), "ncclAllReduce(barrier)");
}

// Copy transport for one exchange step, driven by the host chunk plan
// (exchange_chunks, qvg_schedule.hpp) — the same plan on every transport:
//   * NCCL ranks: chunk i is a grouped ncclSend/ncclRecv with the partner into
//     one of two scratch buffers; its scratch -> shard copy runs on the copy
//     stream and overlaps the send/recv of chunk i+1 (event-ordered; a chunk's
//     copy waits for its own group, so the bytes it overwrites were sent);
//   * virtual shards (one device): chunk i of rank r and chunk i of its
//     partner trade places through a scratch buffer with D2D copies, the
//     pair driven once by its lower rank. The bytes land exactly where the
//     NCCL transport puts them, so the plan runs bit-exactly on one GPU.
inline void copy_exchange(qvg_state &s, ShardSet &set, const ShardStep &step) {
    cudaStream_t st = shard_stream(s);
    const uint32_t S = shard_amp_bytes(s);
    const uint64_t chunk = set.copy_chunk_bytes(S);
    if (set.is_virtual) {
        set.ensure_scratch(chunk);
        for (size_t b = 0; b < set.bufs.size(); ++b) {
            const uint32_t r = set.ranks[b];
            const std::vector<XChunk> mine = exchange_chunks(set.L, S, chunk, r, step);
            std::vector<XChunk> theirs;
            uint32_t cur = ~0u;
            for (size_t i = 0; i < mine.size(); ++i) {
                const XChunk &c = mine[i];
                if (c.partner < r) continue;  // driven by the partner
                if (c.partner != cur) {
                    theirs = exchange_chunks(set.L, S, chunk, c.partner, step);
                    cur = c.partner;
                }
                const XChunk &d = theirs[i];
                if (d.partner != r || d.bytes != c.bytes || d.round != c.round)
                    throw std::runtime_error("internal: exchange chunk plans of a pair disagree");
                char *pa = static_cast<char *>(set.bufs[r]) + c.offset;
                char *pb = static_cast<char *>(set.bufs[c.partner]) + d.offset;
                cuda_throw(cudaMemcpyAsync(set.scratch, pa, c.bytes, cudaMemcpyDeviceToDevice, st), "exchange copy");
                cuda_throw(cudaMemcpyAsync(pa, pb, c.bytes, cudaMemcpyDeviceToDevice, st), "exchange copy");
                cuda_throw(cudaMemcpyAsync(pb, set.scratch, c.bytes, cudaMemcpyDeviceToDevice, st), "exchange copy");
            }
        }
        return;
    }
    const std::vector<XChunk> plan = exchange_chunks(set.L, S, chunk, set.rank, step);
    char *base = static_cast<char *>(set.bufs[0]);
    uint64_t i = 0;
    for (const XChunk &c : plan) {
        char *scr = static_cast<char *>(set.scratch) + (i & 1) * set.chunk_bytes;
        if (i >= 2) cuda_throw(cudaStreamWaitEvent(st, set.copied[i & 1], 0), "wait scratch");
        nccl_check(ncclGroupStart(), "ncclGroupStart");
        nccl_check(ncclSend(base + c.offset, c.bytes, ncclChar, (int)c.partner, set.comm, st), "ncclSend");
        nccl_check(ncclRecv(scr, c.bytes, ncclChar, (int)c.partner, set.comm, st), "ncclRecv");
        nccl_check(ncclGroupEnd(), "ncclGroupEnd");
        cuda_throw(cudaEventRecord(set.received[i & 1], st), "record received");
        cuda_throw(cudaStreamWaitEvent(set.copy_stream, set.received[i & 1], 0), "wait received");
        cuda_throw(cudaMemcpyAsync(base + c.offset, scr, c.bytes, cudaMemcpyDeviceToDevice, set.copy_stream),
                   "exchange copy");
        cuda_throw(cudaEventRecord(set.copied[i & 1], set.copy_stream), "record copied");
        ++i;
    }
    for (int b = 0; b < 2 && (uint64_t)b < i; ++b)  // later work on the state stream sees every copy
        cuda_throw(cudaStreamWaitEvent(st, set.copied[b], 0), "wait copies");
}

// Half-shard exchange swapping global physical qubit gpos with local qubit
// lpos. A rank whose gpos bit is b gives up the amplitudes whose local bit lpos
// is 1-b (2^(L-1-lpos) blocks of 2^lpos contiguous amplitudes) and receives
// the partner's matching half into the same places.
//
// `gate` (or null) is the local step that follows the exchange with its target
// on lpos. The peer and virtual transports apply it inside the exchange kernel
// when the exchange mode asks for it (returns true: the caller drops the
// step). The NCCL copy transport never does.
//
// NCCL copy transport: each block goes in chunks through two scratch buffers.
// The send/recv of chunk i+1 (state stream) overlaps the scratch -> shard copy
// of chunk i (copy stream), ordered by events. A chunk's copy waits for its own
// send/recv group, so the bytes it overwrites were already sent.
inline bool run_exchange(qvg_state &s, ShardSet &set, uint32_t gpos, uint32_t lpos, const ShardStep *gate) {
    cudaStream_t st = shard_stream(s);
    const uint32_t S = shard_amp_bytes(s);
    const uint64_t half = 1ull << (set.L - 1);
    const uint64_t half_bytes = half * S;
    const uint32_t bit = 1u << (gpos - set.L);
    // -1 auto: peer ranks fuse the gate (NVLink-bound, the local bytes are free);
    // virtual shards only exchange (the gate usually joins a fused tile pass).
    int mode = shard_exchange_mode(s);
    if (mode < 0) mode = set.is_virtual ? 1 : 2;
    const bool use_kernel = mode >= 1 && (set.is_virtual || set.peer_ok);
    const bool fuse = use_kernel && mode == 2 && gate != nullptr;
    int cbit = -1, flags = 0;
    const double *u = nullptr;
    auto pred = [&](uint32_t r) { return (r & gate->rank_mask) == gate->rank_value; };
    if (fuse) {
        cbit = gate->op.kind == QVG_OP_CONTROLLED ? gate->op.control : -1;
        u = gate->op.u;
    }
    const bool dbl = S == 16;
    auto xchg = [&](void *a, void *b, uint64_t t0, uint64_t nt, int fl, int fence) {
        if (dbl) launch_xchg<double>(st, a, b, lpos, t0, nt, cbit, fl, u, fence);
        else launch_xchg<float>(st, a, b, lpos, t0, nt, cbit, fl, u, fence);
    };
    const uint64_t quarter = half / 2;  // each rank of a pair streams half of the 2^(L-1) x0's
    qvg_stats &stats = shard_stats(s);
    if (!use_kernel) {  // copy transport (NCCL send/recv, or D2D copies between virtual shards)
        ShardStep xs{};
        xs.type = STEP_EXCHANGE;
        xs.gpos = gpos;
        xs.lpos = lpos;
        copy_exchange(s, set, xs);
        stats.exchanges += 1;
        stats.exchange_bytes += set.is_virtual ? half_bytes * set.world / 2 : half_bytes;
        return false;
    }
    if (set.is_virtual) {
        for (size_t b = 0; b < set.bufs.size(); ++b) {
            const uint32_t r = set.ranks[b];
            if (r & bit) continue;
            const uint32_t partner = r | bit;
            if (fuse) flags = (pred(r) ? 1 : 0) | (pred(partner) ? 2 : 0);
            // one launch per rank role, exactly as the two ranks would split it
            xchg(set.bufs[b], set.bufs[partner], 0, quarter, flags, 0);
            xchg(set.bufs[b], set.bufs[partner], quarter, quarter, flags, 0);
            stats.kernel_launches += 2;
        }
        cuda_throw(cudaGetLastError(), "exchange launch");
        stats.exchanges += 1;
        stats.exchange_bytes += half_bytes * set.world / 2;
        if (fuse) stats.fused_exchanges += 1;
        return fuse;
    }
    const uint32_t partner = set.rank ^ bit;
    if (use_kernel) {
        const bool role_b = (set.rank & bit) != 0;
        void *a = role_b ? set.peer[partner] : set.bufs[0];
        void *b = role_b ? set.bufs[0] : set.peer[partner];
        if (fuse) flags = (pred(set.rank & ~bit) ? 1 : 0) | (pred(set.rank | bit) ? 2 : 0);
        stream_barrier(set, st);  // the partner's earlier passes over its shard are done
        xchg(a, b, role_b ? quarter : 0, quarter, flags, 1);
        cuda_throw(cudaGetLastError(), "exchange launch");
        stream_barrier(set, st);  // both halves are in place before either rank goes on
        stats.kernel_launches += 1;
        stats.exchanges += 1;
        stats.exchange_bytes += half_bytes;
        if (fuse) stats.fused_exchanges += 1;
        return fuse;
    }
    throw std::runtime_error("internal: exchange without a transport");
}

// Batched exchange (STEP_MULTI_EXCHANGE): the 2^k ranks that differ only in
// the swapped rank bits trade, in 2^k - 1 XOR rounds, the regions whose
// local bits at the k positions read the partner's value. Peer and virtual
// transports run all rounds in one k_mxchg launch per rank. The NCCL copy
// transport runs the rounds as pairwise chunked exchanges of those regions.
inline void run_multi_exchange(qvg_state &s, ShardSet &set, const ShardStep &st) {
    cudaStream_t stream = shard_stream(s);
    const uint32_t S = shard_amp_bytes(s);
    const uint32_t k = st.lpos2, mask = st.gpos;
    if (k < 2 || k > 4 || (uint32_t)__builtin_popcount(mask) != k) throw std::runtime_error("internal: bad multi-exchange step");
    int pos[4], idx[4] = {0, 1, 2, 3};
    for (uint32_t i = 0; i < k; ++i) pos[i] = (int)multi_pos(st, i);
    std::sort(idx, idx + k, [&](int a, int b) { return pos[a] < pos[b]; });
    const uint64_t region = 1ull << (set.L - k);  // amplitudes per (rank, partner)
    const uint32_t rounds = (1u << k) - 1;
    qvg_stats &stats = shard_stats(s);
    int mode = shard_exchange_mode(s);
    const bool kernel = mode != 0 && (set.is_virtual || set.peer_ok);
    auto launch = [&](auto tag, void *self, auto &&peer_of, uint32_t w, int fence) {
        using R = decltype(tag);
        using T = typename Cplx<R>::T;
        MxParams<R> p{};
        p.self = static_cast<T *>(self);
        for (uint32_t t = 1; t <= rounds; ++t) p.peer[t] = static_cast<T *>(peer_of(t));
        p.k = (int)k;
        for (uint32_t j = 0; j < k; ++j) {
            p.ps[j] = pos[idx[j]];
            p.perm[j] = idx[j];
        }
        p.w = w;
        p.half = region / 2;
        p.fence = fence;
        if (p.half >= 1024) {
            k_mxchg<R, 4><<<dim3((unsigned)(p.half / 1024), rounds), 256, 0, stream>>>(p);
        } else {
            const unsigned bs = (unsigned)std::min<uint64_t>(p.half, 256);
            k_mxchg<R, 1><<<dim3((unsigned)(p.half / bs), rounds), bs, 0, stream>>>(p);
        }
    };
    auto launch_any = [&](void *self, auto &&peer_of, uint32_t w, int fence) {
        if (S == 16) launch(double{}, self, peer_of, w, fence);
        else launch(float{}, self, peer_of, w, fence);
    };
    const uint32_t gmask = mask;  // rank bits
    if (kernel) {
        if (set.is_virtual) {
            for (size_t b = 0; b < set.bufs.size(); ++b) {
                const uint32_t r = set.ranks[b];
                launch_any(set.bufs[b], [&](uint32_t t) { return set.bufs[r ^ bits_pdep(t, gmask)]; },
                           bits_pext(r, gmask), 0);
                stats.kernel_launches += 1;
            }
            stats.exchange_bytes += (uint64_t)set.world * rounds * region * S;
        } else {
            const uint32_t r = set.rank;
            stream_barrier(set, stream);
            launch_any(set.bufs[0], [&](uint32_t t) { return set.peer[r ^ bits_pdep(t, gmask)]; }, bits_pext(r, gmask),
                       1);
            cuda_throw(cudaGetLastError(), "multi-exchange launch");
            stream_barrier(set, stream);
            stats.kernel_launches += 1;
            stats.exchange_bytes += (uint64_t)rounds * region * S;
        }
        cuda_throw(cudaGetLastError(), "multi-exchange launch");
        stats.exchanges += 1;
        return;
    }
    // copy transport: round t is a pairwise exchange of the region whose
    // local bits read the partner's value (exchange_chunks)
    copy_exchange(s, set, st);
    stats.exchanges += 1;
    stats.exchange_bytes += (set.is_virtual ? set.world : 1) * (uint64_t)rounds * region * S;
}

// Execute a step list: consecutive local steps are batched per shard (each
// shard keeps the ops whose rank predicate it satisfies) and planned together,
// so fusion spans everything between two exchanges. The step right after an
// exchange (the gate that caused it, target on the swapped-in qubit) is offered
// to the exchange kernel.
inline void run_steps(qvg_state &s, ShardSet &set, const std::vector<ShardStep> &steps) {
    std::vector<std::vector<qvg_gate>> batch(set.bufs.size());
    uint64_t segment = 0;
    // One executed segment: hooks before (phase 0) and after its device work
    // completed (phase 1; the stream is synchronised only when a hook is
    // installed), CUDA events around it when timing. A nonzero hook value is
    // an injected fault: IoError, and no later segment runs (the reference's
    // rethrow after join, parallel.cpp:128-132).
    auto run_segment = [&](uint32_t type, auto &&work) {
        const bool hooked = shard_has_hook(s);
        auto call_hooks = [&](uint32_t phase) {
            for (uint32_t r : set.ranks)
                if (shard_step_hook(s, r, segment, type, phase))
                    throw std::runtime_error("injected fault on rank " + std::to_string(r) + " at segment " +
                                             std::to_string(segment) + (phase ? " (end)" : " (start)"));
        };
        if (hooked) call_hooks(0);
        cudaEvent_t ev[2] = {nullptr, nullptr};
        const bool timed = shard_timing(s);
        cudaStream_t st = shard_stream(s);
        if (timed) {
            for (auto &e : ev) cuda_throw(cudaEventCreate(&e), "cudaEventCreate");
            cuda_throw(cudaEventRecord(ev[0], st), "cudaEventRecord");
        }
        work();
        if (timed) {
            cuda_throw(cudaEventRecord(ev[1], st), "cudaEventRecord");
            shard_time_push(s, ev[0], ev[1], (type == STEP_EXCHANGE || type == STEP_MULTI_EXCHANGE) ? 1 : 0);
        }
        if (hooked) {
            cuda_throw(cudaStreamSynchronize(st), "hooked segment sync");
            call_hooks(1);
        }
        ++segment;
    };
    auto flush = [&] {
        bool any = false;
        for (auto &b : batch) any = any || !b.empty();
        if (!any) return;
        run_segment(STEP_LOCAL, [&] {
            for (size_t b = 0; b < set.bufs.size(); ++b) {
                if (!batch[b].empty()) shard_run_local(s, set.bufs[b], batch[b].data(), batch[b].size());
                batch[b].clear();
            }
        });
    };
    for (size_t i = 0; i < steps.size(); ++i) {
        const ShardStep &st = steps[i];
        if (st.type == STEP_LOCAL) {
            for (size_t b = 0; b < set.bufs.size(); ++b)
                if ((set.ranks[b] & st.rank_mask) == st.rank_value) batch[b].push_back(st.op);
            continue;
        }
        flush();
        if (st.type == STEP_EXCHANGE) {
            const ShardStep *next = i + 1 < steps.size() ? &steps[i + 1] : nullptr;
            const bool candidate = next && next->type == STEP_LOCAL && next->op.target == st.lpos &&
                                   !op_is_diag(next->op);
            bool fused = false;
            run_segment(STEP_EXCHANGE, [&] { fused = run_exchange(s, set, st.gpos, st.lpos, candidate ? next : nullptr); });
            if (fused) ++i;
        } else if (st.type == STEP_MULTI_EXCHANGE) {
            run_segment(STEP_MULTI_EXCHANGE, [&] { run_multi_exchange(s, set, st); });
        } else {
            run_segment(STEP_LOCAL_SWAP, [&] { run_local_swap(s, set, st.lpos, st.lpos2); });
        }
    }
    flush();
}

inline void shard_apply(qvg_state &s, ShardSet &set, const qvg_gate *ops, uint64_t count) {
    if (set.world == 1) {
        shard_run_local(s, set.bufs[0], ops, count);
        return;
    }
    std::vector<ShardStep> steps;
    schedule_ops(set.n, set.L, ops, count, set.map, steps, shard_batch_max(s));
    run_steps(s, set, steps);
}

inline void shard_canonicalize(qvg_state &s, ShardSet &set) {
    if (set.world == 1 || set.map.identity()) return;
    std::vector<ShardStep> steps;
    schedule_canonicalize(set.n, set.L, set.map, steps, shard_batch_max(s));
    run_steps(s, set, steps);
}

inline void shard_transfer(qvg_state &s, ShardSet &set, void *host, uint64_t offset, uint64_t count, bool h2d,
                           bool sync = true) {
    shard_canonicalize(s, set);
    cudaStream_t st = shard_stream(s);
    const uint32_t S = shard_amp_bytes(s);
    const uint64_t local = 1ull << set.L;
    for (size_t b = 0; b < set.bufs.size(); ++b) {
        const uint64_t lo = (uint64_t)set.ranks[b] * local, hi = lo + local;
        const uint64_t a = std::max(lo, offset), e = std::min(hi, offset + count);
        if (a >= e) continue;
        char *dev = static_cast<char *>(set.bufs[b]) + (a - lo) * S;
        char *hst = static_cast<char *>(host) + (a - offset) * S;
        if (h2d) cuda_throw(cudaMemcpyAsync(dev, hst, (e - a) * S, cudaMemcpyHostToDevice, st), "H2D");
        else cuda_throw(cudaMemcpyAsync(hst, dev, (e - a) * S, cudaMemcpyDeviceToHost, st), "D2H");
    }
    if (sync) cuda_throw(cudaStreamSynchronize(st), "transfer sync");
}

// Asynchronous NCCL failures (a peer died, a link error) are reported on the
// next qvg_sync as IoError; the whole circuit fails (no elastic recovery, like
// the reference's rethrow-after-join, parallel.cpp:128-132).
inline void shard_check_async(ShardSet &set) {
    if (!set.comm) return;
    ncclResult_t r = ncclSuccess;
    nccl_check(ncclCommGetAsyncError(set.comm, &r), "ncclCommGetAsyncError");
    nccl_check(r, "NCCL asynchronous error");
}

inline double shard_allreduce_op(qvg_state &s, ShardSet &set, double v, ncclRedOp_t op);

inline double shard_allreduce_max(qvg_state &s, ShardSet &set, double v) {
    return shard_allreduce_op(s, set, v, ncclMax);
}

inline double shard_allreduce_sum(qvg_state &s, ShardSet &set, double v) {
    return shard_allreduce_op(s, set, v, ncclSum);
}

inline double shard_allreduce_op(qvg_state &s, ShardSet &set, double v, ncclRedOp_t op) {
    if (!set.comm) return v;
    cudaStream_t st = shard_stream(s);
    cuda_throw(cudaMemcpyAsync(set.d_scalar, &v, sizeof(double), cudaMemcpyHostToDevice, st), "H2D scalar");
    nccl_check(ncclAllReduce(set.d_scalar, set.d_scalar, 1, ncclDouble, op, set.comm, st), "ncclAllReduce");
    double out = 0.0;
    cuda_throw(cudaMemcpyAsync(&out, set.d_scalar, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H scalar");
    cuda_throw(cudaStreamSynchronize(st), "allreduce sync");
    return out;
}

// top_amplitudes (reference engine.cpp:511-544): the k largest |a|^2,
// descending, ties by ascending index — an exact radix select on the device
// (qvg_readout.cuh): six histogram passes over the IEEE bits of |a|^2 find the
// k-th largest key tau, one pass collects the keys above it, and ties at tau
// are taken in index order from the first chunks that hold them. Sharded
// states reduce the histograms with ncclAllReduce and gather the candidates.
inline void shard_top_amplitudes(qvg_state &s, ShardSet &set, uint32_t k, uint64_t *index_out, double *amps_out) {
    if (k == 0) return;
    shard_canonicalize(s, set);
    cudaStream_t st = shard_stream(s);
    const uint32_t S = shard_amp_bytes(s);
    const uint64_t local = 1ull << set.L;
    const uint64_t total = 1ull << set.n;
    const uint32_t kk = (uint32_t)std::min<uint64_t>(k, total);
    const bool dbl = S == 16;
    const unsigned grid = (unsigned)std::min<uint64_t>((local + 255) / 256, 4096);
    // device scratch: histogram (64-bit bins), candidate list, counters
    unsigned long long *d_hist = nullptr;
    unsigned int *d_n = nullptr;
    TopkEntry *d_out = nullptr;
    cuda_throw(cudaMalloc(&d_hist, kTopkBins * sizeof(unsigned long long)), "cudaMalloc(top-k hist)");
    cuda_throw(cudaMalloc(&d_n, sizeof(unsigned int)), "cudaMalloc(top-k count)");
    cuda_throw(cudaMalloc(&d_out, (size_t)kk * sizeof(TopkEntry)), "cudaMalloc(top-k out)");
    struct Free {
        void *p[3];
        ~Free() {
            for (void *q : p) cudaFree(q);
        }
    } guard{{d_hist, d_n, d_out}};
    std::vector<unsigned long long> h(kTopkBins);
    static const int widths[6] = {11, 11, 11, 11, 11, 9};
    uint64_t prefix = 0, needed = kk;
    bool all_above = false;  // every key >= the selected bin's low edge is in
    int shift = 64;
    for (int level = 0; level < 6; ++level) {
        const int w = widths[level];
        shift -= w;
        cuda_throw(cudaMemsetAsync(d_hist, 0, kTopkBins * sizeof(unsigned long long), st), "memset hist");
        for (void *psi : set.bufs) {
            if (dbl) k_topk_hist<double><<<grid, 256, 0, st>>>(static_cast<const double2 *>(psi), local, prefix, shift, w, d_hist);
            else k_topk_hist<float><<<grid, 256, 0, st>>>(static_cast<const float2 *>(psi), local, prefix, shift, w, d_hist);
        }
        cuda_throw(cudaGetLastError(), "top-k hist launch");
        if (set.comm)
            nccl_check(ncclAllReduce(d_hist, d_hist, kTopkBins, ncclUint64, ncclSum, set.comm, st), "ncclAllReduce(hist)");
        cuda_throw(cudaMemcpyAsync(h.data(), d_hist, kTopkBins * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st),
                   "D2H hist");
        cuda_throw(cudaStreamSynchronize(st), "top-k sync");
        uint64_t cum = 0;
        int sel = 0;
        for (int b = (1 << w) - 1; b >= 0; --b) {
            if (cum + h[b] >= needed) {
                sel = b;
                break;
            }
            cum += h[b];
        }
        needed -= cum;
        prefix = (prefix << w) | (uint64_t)sel;
        if (h[sel] == needed) {  // the whole bin is in: no ties to break
            all_above = true;
            break;
        }
    }
    // Collect every key > tau, then fill the remaining kk - |collected| slots
    // with the keys == tie_key in ascending global index.
    //   whole bin in, low edge e > 0: tau = e - 1 (keys >= e), no ties left;
    //   whole bin in, low edge 0 (every key qualifies, e.g. k >= 2^n):
    //     tau = 0 collects the nonzero keys, ties at key 0 fill the rest;
    //   otherwise the full 64-bit key was selected: tau = prefix, ties at tau.
    const uint64_t low_edge = all_above ? prefix << shift : prefix;
    const uint64_t tau = all_above ? (low_edge == 0 ? 0 : low_edge - 1) : prefix;
    const uint64_t tie_key = all_above ? 0 : prefix;
    std::vector<TopkEntry> cand;
    auto gather_rank_lists = [&](std::vector<TopkEntry> &mine) {
        if (!set.comm) return mine;
        // fixed-size allgather of kk entries per rank (index ~0 = empty)
        const size_t per = (size_t)kk * sizeof(TopkEntry);
        std::vector<TopkEntry> pad(kk, TopkEntry{~0ull, 0.0, 0.0});
        std::copy(mine.begin(), mine.begin() + std::min<size_t>(mine.size(), kk), pad.begin());
        char *d = nullptr;
        cuda_throw(cudaMalloc(&d, per * (set.world + 1)), "cudaMalloc(top-k gather)");
        cuda_throw(cudaMemcpyAsync(d, pad.data(), per, cudaMemcpyHostToDevice, st), "H2D");
        nccl_check(ncclAllGather(d, d + per, per, ncclChar, set.comm, st), "ncclAllGather(top-k)");
        std::vector<TopkEntry> all((size_t)kk * set.world);
        cuda_throw(cudaMemcpyAsync(all.data(), d + per, per * set.world, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_throw(cudaStreamSynchronize(st), "gather sync");
        cudaFree(d);
        std::vector<TopkEntry> out;
        for (const TopkEntry &e : all)
            if (e.index != ~0ull) out.push_back(e);
        return out;
    };
    {
        cuda_throw(cudaMemsetAsync(d_n, 0, sizeof(unsigned int), st), "memset count");
        for (size_t b = 0; b < set.bufs.size(); ++b) {
            const uint64_t base = (uint64_t)set.ranks[b] * local;
            if (dbl) k_topk_collect<double><<<grid, 256, 0, st>>>(static_cast<const double2 *>(set.bufs[b]), local, base, tau, d_out, d_n, kk);
            else k_topk_collect<float><<<grid, 256, 0, st>>>(static_cast<const float2 *>(set.bufs[b]), local, base, tau, d_out, d_n, kk);
        }
        cuda_throw(cudaGetLastError(), "top-k collect launch");
        unsigned int n_out = 0;
        cuda_throw(cudaMemcpyAsync(&n_out, d_n, sizeof(n_out), cudaMemcpyDeviceToHost, st), "D2H count");
        cuda_throw(cudaStreamSynchronize(st), "top-k sync");
        std::vector<TopkEntry> mine(std::min<unsigned int>(n_out, kk));
        if (!mine.empty())
            cuda_throw(cudaMemcpy(mine.data(), d_out, mine.size() * sizeof(TopkEntry), cudaMemcpyDeviceToHost), "D2H");
        cand = gather_rank_lists(mine);
    }
    needed = cand.size() < kk ? kk - cand.size() : 0;
    if (needed > 0) {  // ties at tie_key, by ascending global index
        constexpr uint64_t chunk = 1ull << 16;
        const uint64_t nchunks = (local + chunk - 1) / chunk;
        unsigned int *d_cnt = nullptr;
        unsigned char *d_flags = nullptr;
        cuda_throw(cudaMalloc(&d_cnt, nchunks * sizeof(unsigned int)), "cudaMalloc(tie counts)");
        cuda_throw(cudaMalloc(&d_flags, chunk), "cudaMalloc(tie flags)");
        std::vector<TopkEntry> ties;
        std::vector<unsigned int> cnt(nchunks);
        std::vector<unsigned char> flags(chunk);
        std::vector<char> host((size_t)chunk * S);
        for (size_t b = 0; b < set.bufs.size() && ties.size() < needed; ++b) {
            if (dbl) k_topk_tie_counts<double><<<(unsigned)nchunks, 256, 0, st>>>(static_cast<const double2 *>(set.bufs[b]), local, chunk, tie_key, d_cnt);
            else k_topk_tie_counts<float><<<(unsigned)nchunks, 256, 0, st>>>(static_cast<const float2 *>(set.bufs[b]), local, chunk, tie_key, d_cnt);
            cuda_throw(cudaGetLastError(), "tie count launch");
            cuda_throw(cudaMemcpyAsync(cnt.data(), d_cnt, nchunks * sizeof(unsigned int), cudaMemcpyDeviceToHost, st), "D2H");
            cuda_throw(cudaStreamSynchronize(st), "tie sync");
            const uint64_t base = (uint64_t)set.ranks[b] * local;
            for (uint64_t c = 0; c < nchunks && ties.size() < needed; ++c) {
                if (!cnt[c]) continue;
                const uint64_t len = std::min(chunk, local - c * chunk);
                if (dbl) k_topk_tie_flags<double><<<64, 256, 0, st>>>(static_cast<const double2 *>(set.bufs[b]), c * chunk, len, tie_key, d_flags);
                else k_topk_tie_flags<float><<<64, 256, 0, st>>>(static_cast<const float2 *>(set.bufs[b]), c * chunk, len, tie_key, d_flags);
                cuda_throw(cudaGetLastError(), "tie flags launch");
                cuda_throw(cudaMemcpyAsync(flags.data(), d_flags, len, cudaMemcpyDeviceToHost, st), "D2H tie flags");
                cuda_throw(cudaMemcpyAsync(host.data(), static_cast<char *>(set.bufs[b]) + c * chunk * S, len * S,
                                           cudaMemcpyDeviceToHost, st), "D2H tie chunk");
                cuda_throw(cudaStreamSynchronize(st), "tie chunk sync");
                for (uint64_t j = 0; j < len && ties.size() < needed; ++j) {
                    if (!flags[j]) continue;
                    double re, im;
                    if (dbl) {
                        re = reinterpret_cast<const double *>(host.data())[2 * j];
                        im = reinterpret_cast<const double *>(host.data())[2 * j + 1];
                    } else {
                        re = reinterpret_cast<const float *>(host.data())[2 * j];
                        im = reinterpret_cast<const float *>(host.data())[2 * j + 1];
                    }
                    ties.push_back(TopkEntry{base + c * chunk + j, re, im});
                }
            }
        }
        cudaFree(d_cnt);
        cudaFree(d_flags);
        // sharded: every rank offers its first ties; the lowest indices win below
        std::vector<TopkEntry> all_ties = gather_rank_lists(ties);
        cand.insert(cand.end(), all_ties.begin(), all_ties.end());
    }
    // |a|^2 without FMA contraction (volatile products), so the host orders
    // candidates by the same rounded keys the device selected on
    auto prob = [](const TopkEntry &e) {
        volatile double rr = e.re * e.re, ii = e.im * e.im;
        return rr + ii;
    };
    std::sort(cand.begin(), cand.end(), [&](const TopkEntry &a, const TopkEntry &b) {
        const double pa = prob(a), pb = prob(b);
        return pa != pb ? pa > pb : a.index < b.index;
    });
    for (uint32_t j = 0; j < k; ++j) {
        if (j < cand.size() && j < kk) {
            index_out[j] = cand[j].index;
            amps_out[2 * j] = cand[j].re;
            amps_out[2 * j + 1] = cand[j].im;
        } else {
            index_out[j] = ~0ull;
            amps_out[2 * j] = amps_out[2 * j + 1] = 0.0;
        }
    }
}
}  // namespace qvg
