// qvg_shard.hpp — state sharding over G = 2^g GPUs, executing
// the host schedule of qvg_schedule.hpp.
//
// Two transports behind one executor:
//   * NCCL (one process per GPU, the deployment mode): a global-target gate
//     triggers a pairwise half-shard exchange with ncclSend/ncclRecv over
//     NVLink, chunked through a scratch buffer;
//   * virtual shards (all G shards on this device, one process): the same
//     schedule with exchanges done as device-side range swaps. This is how the
//     sharded path is tested bit-for-bit on a single GPU (the profiling guide
//     forbids emulating ranks as processes that wait on each other).
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
#include "qvg_schedule.hpp"

struct qvg_state;

namespace qvg {

// Hooks implemented in qvg_engine.cu.
void shard_run_local(qvg_state &s, void *psi, const qvg_gate *ops, uint64_t count);
cudaStream_t shard_stream(qvg_state &s);
uint32_t shard_amp_bytes(const qvg_state &s);
qvg_stats &shard_stats(qvg_state &s);
void cuda_throw(cudaError_t e, const char *what);

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
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t received[2] = {nullptr, nullptr}, copied[2] = {nullptr, nullptr};
    double *d_scalar = nullptr;

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
        }
    }

    void release() {
        for (void *p : bufs) cudaFree(p);
        bufs.clear();
        ranks.clear();
        if (scratch) cudaFree(scratch);
        scratch = nullptr;
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

// Virtual-shard exchange: p's amplitudes with local bit lpos = 1 trade places
// with q's amplitudes with local bit lpos = 0.
template <class R>
inline void launch_swap_halves(cudaStream_t st, void *p, void *q, uint32_t L, uint32_t lpos) {
    using T = typename Cplx<R>::T;
    const uint64_t count = 1ull << (L - 1);
    if (count >= 1024)
        k_swap_halves<R, 4><<<(unsigned)(count / 1024), 256, 0, st>>>(static_cast<T *>(p), static_cast<T *>(q),
                                                                       (int)lpos);
    else {
        const unsigned bs = (unsigned)std::min<uint64_t>(count, 256);
        k_swap_halves<R, 1><<<(unsigned)(count / bs), bs, 0, st>>>(static_cast<T *>(p), static_cast<T *>(q),
                                                                    (int)lpos);
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

// Half-shard exchange swapping global physical qubit gpos with local qubit
// lpos: a rank whose gpos bit is b sends the amplitudes whose local bit lpos is
// 1-b (2^(L-1-lpos) blocks of 2^lpos contiguous amplitudes) and receives the
// partner's matching half into the same places.
//
// NCCL transport: each block goes in chunks through two scratch buffers; the
// send/recv of chunk i+1 (state stream) overlaps the scratch -> shard copy of
// chunk i (copy stream), ordered by events. A chunk's copy waits for its own
// send/recv group, so the bytes it overwrites were already sent.
inline void run_exchange(qvg_state &s, ShardSet &set, uint32_t gpos, uint32_t lpos) {
    cudaStream_t st = shard_stream(s);
    const uint32_t S = shard_amp_bytes(s);
    const uint64_t half = 1ull << (set.L - 1);
    const uint64_t half_bytes = half * S;
    const uint32_t bit = 1u << (gpos - set.L);
    if (set.is_virtual) {
        for (size_t b = 0; b < set.bufs.size(); ++b) {
            const uint32_t r = set.ranks[b];
            if (r & bit) continue;
            const uint32_t partner = r | bit;
            // r (bit 0) sends its lpos=1 half; partner (bit 1) its lpos=0 half.
            if (S == 16) launch_swap_halves<double>(st, set.bufs[b], set.bufs[partner], set.L, lpos);
            else launch_swap_halves<float>(st, set.bufs[b], set.bufs[partner], set.L, lpos);
        }
        cuda_throw(cudaGetLastError(), "exchange launch");
        shard_stats(s).exchanges += 1;
        shard_stats(s).exchange_bytes += half_bytes * set.world / 2;
        return;
    }
    const int partner = (int)(set.rank ^ bit);
    const uint64_t sendbit = (set.rank & bit) ? 0 : 1;  // my half: local bit lpos == sendbit
    const uint64_t block_bytes = (uint64_t)S << lpos;
    const uint64_t nblocks = 1ull << (set.L - 1 - lpos);
    char *base = static_cast<char *>(set.bufs[0]);
    uint64_t i = 0;
    for (uint64_t k = 0; k < nblocks; ++k) {
        char *blk = base + (((k << 1) | sendbit) * block_bytes);
        for (uint64_t off = 0; off < block_bytes; off += set.chunk_bytes, ++i) {
            const uint64_t c = std::min<uint64_t>(set.chunk_bytes, block_bytes - off);
            char *scr = static_cast<char *>(set.scratch) + (i & 1) * set.chunk_bytes;
            if (i >= 2) cuda_throw(cudaStreamWaitEvent(st, set.copied[i & 1], 0), "wait scratch");
            nccl_check(ncclGroupStart(), "ncclGroupStart");
            nccl_check(ncclSend(blk + off, c, ncclChar, partner, set.comm, st), "ncclSend");
            nccl_check(ncclRecv(scr, c, ncclChar, partner, set.comm, st), "ncclRecv");
            nccl_check(ncclGroupEnd(), "ncclGroupEnd");
            cuda_throw(cudaEventRecord(set.received[i & 1], st), "record received");
            cuda_throw(cudaStreamWaitEvent(set.copy_stream, set.received[i & 1], 0), "wait received");
            cuda_throw(cudaMemcpyAsync(blk + off, scr, c, cudaMemcpyDeviceToDevice, set.copy_stream), "exchange copy");
            cuda_throw(cudaEventRecord(set.copied[i & 1], set.copy_stream), "record copied");
        }
    }
    for (int b = 0; b < 2 && (uint64_t)b < i; ++b)  // later work on the state stream sees every copy
        cuda_throw(cudaStreamWaitEvent(st, set.copied[b], 0), "wait copies");
    shard_stats(s).exchanges += 1;
    shard_stats(s).exchange_bytes += half_bytes;
}

// Execute a step list: consecutive local steps are batched per shard (each
// shard keeps the ops whose rank predicate it satisfies) and planned together,
// so fusion spans everything between two exchanges.
inline void run_steps(qvg_state &s, ShardSet &set, const std::vector<ShardStep> &steps) {
    std::vector<std::vector<qvg_gate>> batch(set.bufs.size());
    auto flush = [&] {
        for (size_t b = 0; b < set.bufs.size(); ++b) {
            if (!batch[b].empty()) shard_run_local(s, set.bufs[b], batch[b].data(), batch[b].size());
            batch[b].clear();
        }
    };
    for (const ShardStep &st : steps) {
        if (st.type == STEP_LOCAL) {
            for (size_t b = 0; b < set.bufs.size(); ++b)
                if ((set.ranks[b] & st.rank_mask) == st.rank_value) batch[b].push_back(st.op);
            continue;
        }
        flush();
        if (st.type == STEP_EXCHANGE) run_exchange(s, set, st.gpos, st.lpos);
        else run_local_swap(s, set, st.lpos, st.lpos2);
    }
    flush();
}

inline void shard_apply(qvg_state &s, ShardSet &set, const qvg_gate *ops, uint64_t count) {
    if (set.world == 1) {
        shard_run_local(s, set.bufs[0], ops, count);
        return;
    }
    std::vector<ShardStep> steps;
    schedule_ops(set.n, set.L, ops, count, set.map, steps);
    run_steps(s, set, steps);
}

inline void shard_canonicalize(qvg_state &s, ShardSet &set) {
    if (set.world == 1 || set.map.identity()) return;
    std::vector<ShardStep> steps;
    schedule_canonicalize(set.n, set.L, set.map, steps);
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

inline double shard_allreduce_sum(qvg_state &s, ShardSet &set, double v) {
    if (!set.comm) return v;
    cudaStream_t st = shard_stream(s);
    cuda_throw(cudaMemcpyAsync(set.d_scalar, &v, sizeof(double), cudaMemcpyHostToDevice, st), "H2D scalar");
    nccl_check(ncclAllReduce(set.d_scalar, set.d_scalar, 1, ncclDouble, ncclSum, set.comm, st), "ncclAllReduce");
    double out = 0.0;
    cuda_throw(cudaMemcpyAsync(&out, set.d_scalar, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H scalar");
    cuda_throw(cudaStreamSynchronize(st), "allreduce sync");
    return out;
}

// top_amplitudes (reference engine.cpp:511-544): the k largest |a|^2,
// descending, ties by ascending index. Streams the shard through a chunked
// D2H copy and keeps a k-heap on the host.
inline void shard_top_amplitudes(qvg_state &s, ShardSet &set, uint32_t k, uint64_t *index_out, double *amps_out) {
    if (k == 0) return;
    shard_canonicalize(s, set);
    cudaStream_t st = shard_stream(s);
    const uint32_t S = shard_amp_bytes(s);
    struct Entry {
        double p;
        uint64_t i;
        double re, im;
    };
    auto better = [](const Entry &a, const Entry &b) { return a.p != b.p ? a.p > b.p : a.i < b.i; };
    std::priority_queue<Entry, std::vector<Entry>, decltype(better)> heap(better);
    const uint64_t local = 1ull << set.L;
    const uint64_t chunk = std::min<uint64_t>(local, 1ull << 22);
    std::vector<double> host(chunk * 2);
    std::vector<float> hostf(S == 8 ? chunk * 2 : 0);
    for (size_t b = 0; b < set.bufs.size(); ++b) {
        const uint64_t base = (uint64_t)set.ranks[b] * local;
        for (uint64_t off = 0; off < local; off += chunk) {
            void *dst = S == 16 ? (void *)host.data() : (void *)hostf.data();
            cuda_throw(cudaMemcpyAsync(dst, static_cast<char *>(set.bufs[b]) + off * S, chunk * S,
                                       cudaMemcpyDeviceToHost, st),
                       "top-k D2H");
            cuda_throw(cudaStreamSynchronize(st), "top-k sync");
            for (uint64_t j = 0; j < chunk; ++j) {
                const double re = S == 16 ? host[2 * j] : (double)hostf[2 * j];
                const double im = S == 16 ? host[2 * j + 1] : (double)hostf[2 * j + 1];
                const Entry e{re * re + im * im, base + off + j, re, im};
                if (heap.size() < k) heap.push(e);
                else if (better(e, heap.top())) {
                    heap.pop();
                    heap.push(e);
                }
            }
        }
    }
    std::vector<Entry> all;
    while (!heap.empty()) {
        all.push_back(heap.top());
        heap.pop();
    }
    if (set.comm) {
        // Gather every rank's k candidates (padded) and re-select.
        std::vector<double> mine(4 * (size_t)k, 0.0);
        for (size_t j = 0; j < all.size(); ++j) {
            mine[4 * j] = all[j].p;
            std::memcpy(&mine[4 * j + 1], &all[j].i, sizeof(uint64_t));
            mine[4 * j + 2] = all[j].re;
            mine[4 * j + 3] = all[j].im;
        }
        for (size_t j = all.size(); j < k; ++j) mine[4 * j] = -1.0;
        double *d = nullptr;
        const size_t per = 4 * (size_t)k;
        cuda_throw(cudaMalloc(&d, per * (set.world + 1) * sizeof(double)), "cudaMalloc(top-k gather)");
        cuda_throw(cudaMemcpyAsync(d, mine.data(), per * sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
        nccl_check(ncclAllGather(d, d + per, per, ncclDouble, set.comm, st), "ncclAllGather");
        std::vector<double> gathered(per * set.world);
        cuda_throw(cudaMemcpyAsync(gathered.data(), d + per, gathered.size() * sizeof(double),
                                   cudaMemcpyDeviceToHost, st),
                   "D2H");
        cuda_throw(cudaStreamSynchronize(st), "top-k gather sync");
        cudaFree(d);
        all.clear();
        for (size_t j = 0; j < (size_t)k * set.world; ++j) {
            if (gathered[4 * j] < 0) continue;
            Entry e;
            e.p = gathered[4 * j];
            std::memcpy(&e.i, &gathered[4 * j + 1], sizeof(uint64_t));
            e.re = gathered[4 * j + 2];
            e.im = gathered[4 * j + 3];
            all.push_back(e);
        }
    }
    std::sort(all.begin(), all.end(), better);
    for (uint32_t j = 0; j < k; ++j) {
        if (j < all.size()) {
            index_out[j] = all[j].i;
            amps_out[2 * j] = all[j].re;
            amps_out[2 * j + 1] = all[j].im;
        } else {
            index_out[j] = ~0ull;
            amps_out[2 * j] = amps_out[2 * j + 1] = 0.0;
        }
    }
}

}  // namespace qvg
