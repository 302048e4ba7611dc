// qvg_tile_pipe.cuh — K4b, the fused tile pass as a warp-specialised
// producer/consumer pipeline (VERDICT r1 "next" #4): the same register-group op
// loop as k_tile (qvg_tile.cuh), but tiles move between HBM and shared memory
// with bulk asynchronous copies instead of per-thread 16-B loads and stores.
//
// CTA = 4 consumer warps (128 threads, one 2^SUB-amplitude register subcube
// each, exactly k_tile's 128-thread layout) + 1 producer warp. The CTA is
// persistent over tiles blockIdx.x, blockIdx.x + gridDim.x, ... and keeps a
// ring of STAGES tile slots in shared memory:
//
//   producer, tile i (slot s = i % STAGES):
//     wait done[s] (consumers finished tile i - STAGES and wrote it to s)
//     cp.async.bulk shared -> global of tile i - STAGES, one copy per
//       contiguous segment (2^lowc amplitudes), bulk_group;
//       cp.async.bulk.wait_group.read 0 (the slot's bytes have left)
//     mbarrier.arrive.expect_tx(full[s], tile bytes)
//     cp.async.bulk global -> shared of tile i, complete_tx on full[s]
//   consumers, tile i:
//     wait full[s]; run the register groups (the slot doubles as the
//     transpose buffer between groups); write the result into the slot;
//     fence.proxy.async (generic writes -> the bulk store's async reads);
//     mbarrier.arrive(done[s])
//
// So HBM reads of tiles i+1 .. i+STAGES-1 and the write of tile i-1 are in
// flight while tile i computes, with no registers spent on loads in flight
// (the reason every register/cp.async prefetch of round 1 lost to occupancy).
//
// Slot layout: the bulk copies land the tile linearly (segment h at
// h * 2^lowc amplitudes, local index l at l). Intermediate groups use the
// swizzled layout swz(l) of k_tile (conflict-free transposes). A group whose
// lanes would stride through the linear layout (the planner's "staged" first
// / last groups, which hold tile bits 0..2) moves through it coalesced
// (index t + j*128) and transposes through the swizzled layout, as k_tile does
// through HBM. Layout changes inside one slot need a consumer barrier first
// (named barrier 1, 128 threads); same-layout rewrites do not, because each
// thread rewrites exactly the slots it read.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "qvg_tile.cuh"

namespace qvg {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}
// global -> shared, completion counted in bytes on the mbarrier
__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
// shared -> global, tracked by this thread's bulk groups
__device__ __forceinline__ void bulk_store(void *dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// consumers only (the producer warp never joins): named barrier 1, 128 threads
__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

constexpr int kPipeConsumers = 128;
constexpr int kPipeThreads = kPipeConsumers + 32;

// Shared memory of k_tile_pipe: the high-qubit offset table, 2*STAGES
// mbarriers, then the ring (128-B aligned slots).
__host__ __device__ constexpr uint32_t pipe_ring_offset(int nhi, int stages) {
    return (((8u << nhi) + 16u * (uint32_t)stages) + 127u) & ~127u;
}
__host__ __device__ constexpr uint32_t pipe_smem_bytes(int nhi, int k, int amp_bytes, int stages) {
    return pipe_ring_offset(nhi, stages) + (uint32_t)stages * ((uint32_t)amp_bytes << k);
}

#ifndef QVG_PIPE_MINB
#define QVG_PIPE_MINB 3  // CTAs/SM: 3 x (2 x 32 KB ring + 2 KB) fits 227 KB; 136 registers/thread
#endif

template <class R, int SUB, bool FMA, int CM, int STAGES>
__global__ void __launch_bounds__(kPipeThreads, QVG_PIPE_MINB)
k_tile_pipe(typename Cplx<R>::T *__restrict__ psi, const __grid_constant__ TileParams prm) {
    using T = typename Cplx<R>::T;
    constexpr int E = 1 << SUB;
    constexpr uint32_t NC = kPipeConsumers;
    const TileGeom &g = prm.g;
    const TileOp *ops = prm.ops;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *offhi = reinterpret_cast<uint64_t *>(smem_raw);
    const uint32_t bar0 = smem_u32(smem_raw + (8u << g.nhi));  // full[s] at bar0 + 8s, done[s] at bar0 + 8(STAGES+s)
    T *ring = reinterpret_cast<T *>(smem_raw + pipe_ring_offset(g.nhi, STAGES));
    const uint32_t tile_amps = 1u << g.k;
    const uint32_t nhi = 1u << g.nhi;
    const uint32_t lowm = (1u << g.lowc) - 1u;
    for (uint32_t h = threadIdx.x; h < nhi; h += blockDim.x) {
        uint64_t off = 0;
#pragma unroll
        for (int i = 0; i < 24; ++i)
            if (i < g.nhi && ((h >> i) & 1u)) off |= 1ull << g.hiq[i];
        offhi[h] = off;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(bar0 + 8u * s, 1);                            // full: the producer's expect_tx arrival
            mbar_init(bar0 + 8u * (STAGES + s), NC);                // done: every consumer thread
        }
        fence_mbar_init();
    }
    __syncthreads();
    auto tile_base = [&](uint64_t tile) {
        uint64_t base = tile << g.lowc;
#pragma unroll
        for (int i = 0; i < 24; ++i)
            if (i < g.nhi) base = ins0(base, g.hiq[i]);
        return base;
    };
    const uint64_t first = blockIdx.x;
    const uint64_t cnt = first < g.ntiles ? (g.ntiles - first + gridDim.x - 1) / gridDim.x : 0;

    if (threadIdx.x >= NC) {  // ---------------- producer warp ----------------
        const uint32_t lane = threadIdx.x & 31u;
        const uint32_t seg_bytes = (uint32_t)sizeof(T) << g.lowc;
        const uint32_t seg_amps = 1u << g.lowc;
        auto store_tile = [&](uint64_t i) {  // slot i % STAGES -> HBM (tile i)
            const uint32_t s = (uint32_t)(i % STAGES);
            mbar_wait(bar0 + 8u * (STAGES + s), (uint32_t)((i / STAGES) & 1));
            const uint64_t base = tile_base(first + i * gridDim.x);
            const uint32_t slot = smem_u32(ring + (size_t)s * tile_amps);
            for (uint32_t h = lane; h < nhi; h += 32)
                bulk_store(psi + (base | offhi[h]), slot + h * seg_bytes, seg_bytes);
            bulk_commit();
        };
        for (uint64_t i = 0; i < cnt; ++i) {
            const uint32_t s = (uint32_t)(i % STAGES);
            if (i >= STAGES) {
                store_tile(i - STAGES);
                bulk_wait_read0();  // this lane's stores have read the slot
            }
            __syncwarp();
            const uint32_t full = bar0 + 8u * s;
            if (lane == 0) mbar_expect_tx(full, (uint32_t)sizeof(T) * tile_amps);
            __syncwarp();
            const uint64_t base = tile_base(first + i * gridDim.x);
            const uint32_t slot = smem_u32(ring + (size_t)s * tile_amps);
            for (uint32_t h = lane; h < nhi; h += 32)
                bulk_load(slot + h * seg_bytes, psi + (base | offhi[h]), seg_bytes, full);
            (void)seg_amps;
        }
        for (uint64_t i = cnt > STAGES ? cnt - STAGES : 0; i < cnt; ++i) store_tile(i);
        bulk_wait0();  // every store complete before the CTA's shared memory goes away
        return;
    }

    // ---------------- consumer warps ----------------
    const uint32_t t = threadIdx.x;
    for (uint64_t i = 0; i < cnt; ++i) {
        const uint32_t s = (uint32_t)(i % STAGES);
        const uint64_t base = tile_base(first + i * gridDim.x);
        T *sm = ring + (size_t)s * tile_amps;
        mbar_wait(bar0 + 8u * s, (uint32_t)((i / STAGES) & 1));
        int rec = 0;
        bool linear = true;  // the layout the slot currently holds (this thread's slots)
        for (int gi = 0; gi < g.ngroups; ++gi) {
            const int nops = ops[rec].tbit;
            const uint64_t packed = ops[rec].gtgt;
            ++rec;
            int b[SUB];
#pragma unroll
            for (int j = 0; j < SUB; ++j) b[j] = (int)((packed >> (8 * j)) & 0xff);
            uint32_t l0 = t;
#pragma unroll
            for (int j = 0; j < SUB; ++j) l0 = (uint32_t)ins0(l0, b[j]);
            auto lidx = [&](int r) {
                uint32_t l = l0;
#pragma unroll
                for (int j = 0; j < SUB; ++j) l |= ((r >> j) & 1) ? (1u << b[j]) : 0u;
                return l;
            };
            T v[E];
            if (gi == 0 && (g.stage & 1)) {
                // lanes of this group would stride through the linear slot:
                // read it coalesced, transpose through the swizzled layout
#pragma unroll
                for (int j = 0; j < E; ++j) v[j] = sm[t + (uint32_t)j * NC];
                cbar();
#pragma unroll
                for (int j = 0; j < E; ++j) sm[swz(t + (uint32_t)j * NC)] = v[j];
                cbar();
#pragma unroll
                for (int r = 0; r < E; ++r) v[r] = sm[swz(lidx(r))];
                linear = false;
            } else if (gi == 0) {
#pragma unroll
                for (int r = 0; r < E; ++r) v[r] = sm[lidx(r)];
            } else {
#pragma unroll
                for (int r = 0; r < E; ++r) v[r] = sm[swz(lidx(r))];
            }
            for (int k = 0; k < nops; ++k) {
                const TileOp &op = ops[rec + k];
                if ((base & op.greq) != op.greq) continue;  // control outside the tile is 0
                const int sl = op.slot;
                if ((sl & kSlotCtlTest) && !((t >> op.cbit) & 1u)) continue;
                bool t1 = false;
                if (sl & kSlotT1) t1 = op.tbit >= 0 ? ((t >> op.tbit) & 1u) != 0 : (base & op.gtgt) != 0;
                op_dispatch<R, SUB, FMA, CM>(sl & 0xff, v, reinterpret_cast<const R *>(op.u), t1, (sl & kSlotD0) != 0);
            }
            rec += nops;
            if (gi == g.ngroups - 1) {
                if (g.stage & 2) {
                    // leave coalesced: group layout -> swizzled -> linear
                    if (linear) cbar();
#pragma unroll
                    for (int r = 0; r < E; ++r) sm[swz(lidx(r))] = v[r];
                    cbar();
#pragma unroll
                    for (int j = 0; j < E; ++j) v[j] = sm[swz(t + (uint32_t)j * NC)];
                    cbar();
#pragma unroll
                    for (int j = 0; j < E; ++j) sm[t + (uint32_t)j * NC] = v[j];
                } else {
                    if (!linear) cbar();
#pragma unroll
                    for (int r = 0; r < E; ++r) sm[lidx(r)] = v[r];
                }
                fence_proxy_async();                 // generic writes -> the bulk store's reads
                mbar_arrive(bar0 + 8u * (STAGES + s));
            } else {
                if (linear) cbar();  // others may still read the linear layout here
#pragma unroll
                for (int r = 0; r < E; ++r) sm[swz(lidx(r))] = v[r];
                cbar();
                linear = false;
            }
        }
    }
}

// ---- K4c: the same pipeline with ONE tensor-map TMA per tile -------------------
// k_tile_pipe issues a bulk copy per contiguous segment, and cp.async.bulk takes
// uniform operands, so the producer walks its lanes' segments through an R2UR
// waterfall: 512 serialised trips per tile of 256 x 128-B segments
// (profiles/r02_pipe_sass.txt). Here the tile is one box of a <= 5-D tensor
// map (TileTma, built per pass on the host): one cp.async.bulk.tensor load and
// one store per tile. The map uses SWIZZLE_128B, whose layout in a 1024-B
// aligned slot is exactly k_tile's swizzled layout swz(l) (16-B column ^=
// 128-B row index & 7), so consumers read and write every group through
// swz(lidx) with no staging transposes and no bank conflicts, and the TMA
// store un-swizzles on the way out.
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap *map, const int (&c)[5], uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_store_5d(const CUtensorMap *map, const int (&c)[5], uint32_t src) {
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(src)
                 : "memory");
}

__host__ __device__ constexpr uint32_t tma_ring_offset(int stages) { return (16u * (uint32_t)stages + 1023u) & ~1023u; }
__host__ __device__ constexpr uint32_t tma_smem_bytes(int k, int amp_bytes, int stages) {
    return tma_ring_offset(stages) + (uint32_t)stages * ((uint32_t)amp_bytes << k) + 1024u;  // + slack to 1024-align
}

template <class R, int SUB, bool FMA, int CM, int STAGES>
__global__ void __launch_bounds__(kPipeThreads, QVG_PIPE_MINB)
k_tile_tma(typename Cplx<R>::T *__restrict__ psi, const __grid_constant__ TileParams prm) {
    using T = typename Cplx<R>::T;
    constexpr int E = 1 << SUB;
    constexpr uint32_t NC = kPipeConsumers;
    const TileGeom &g = prm.g;
    const TileOp *ops = prm.ops;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-B aligned ring (SWIZZLE_128B atoms), mbarriers below it
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t pad = ((raw + 1023u) & ~1023u) - raw;
    unsigned char *base_ptr = smem_raw + pad;
    const uint32_t bar0 = smem_u32(base_ptr);  // full[s] at bar0 + 8s, done[s] at bar0 + 8(STAGES+s)
    T *ring = reinterpret_cast<T *>(base_ptr + tma_ring_offset(STAGES));
    const uint32_t tile_amps = 1u << g.k;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(bar0 + 8u * s, 1);
            mbar_init(bar0 + 8u * (STAGES + s), NC);
        }
        fence_mbar_init();
    }
    __syncthreads();
    auto tile_base = [&](uint64_t tile) {
        uint64_t base = tile << g.lowc;
#pragma unroll
        for (int i = 0; i < 24; ++i)
            if (i < g.nhi) base = ins0(base, g.hiq[i]);
        return base;
    };
    const uint64_t first = blockIdx.x;
    const uint64_t cnt = first < g.ntiles ? (g.ntiles - first + gridDim.x - 1) / gridDim.x : 0;

    if (threadIdx.x >= NC) {  // ---------------- producer warp (one lane) ----------------
        if ((threadIdx.x & 31u) != 0) return;
        const CUtensorMap *map = &prm.tma.map;
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
        auto coords = [&](uint64_t tile, int(&c)[5]) {
            const uint64_t base = tile_base(tile);
            c[0] = 0;
#pragma unroll
            for (int d = 1; d < 5; ++d)
                c[d] = prm.tma.gap[d] ? (int)((base >> prm.tma.shift[d]) & ((1ull << prm.tma.len[d]) - 1)) : 0;
        };
        auto store_tile = [&](uint64_t i) {
            const uint32_t s = (uint32_t)(i % STAGES);
            mbar_wait(bar0 + 8u * (STAGES + s), (uint32_t)((i / STAGES) & 1));
            int c[5];
            coords(first + i * gridDim.x, c);
            tma_store_5d(map, c, smem_u32(ring + (size_t)s * tile_amps));
            bulk_commit();
        };
        for (uint64_t i = 0; i < cnt; ++i) {
            const uint32_t s = (uint32_t)(i % STAGES);
            if (i >= STAGES) {
                store_tile(i - STAGES);
                bulk_wait_read0();
            }
            const uint32_t full = bar0 + 8u * s;
            mbar_expect_tx(full, (uint32_t)sizeof(T) * tile_amps);
            int c[5];
            coords(first + i * gridDim.x, c);
            tma_load_5d(smem_u32(ring + (size_t)s * tile_amps), map, c, full);
        }
        for (uint64_t i = cnt > STAGES ? cnt - STAGES : 0; i < cnt; ++i) store_tile(i);
        bulk_wait0();
        return;
    }

    // ---------------- consumer warps: every group through swz(lidx) ----------------
    const uint32_t t = threadIdx.x;
    for (uint64_t i = 0; i < cnt; ++i) {
        const uint32_t s = (uint32_t)(i % STAGES);
        const uint64_t base = tile_base(first + i * gridDim.x);
        T *sm = ring + (size_t)s * tile_amps;
        mbar_wait(bar0 + 8u * s, (uint32_t)((i / STAGES) & 1));
        int rec = 0;
        for (int gi = 0; gi < g.ngroups; ++gi) {
            const int nops = ops[rec].tbit;
            const uint64_t packed = ops[rec].gtgt;
            ++rec;
            int b[SUB];
#pragma unroll
            for (int j = 0; j < SUB; ++j) b[j] = (int)((packed >> (8 * j)) & 0xff);
            uint32_t l0 = t;
#pragma unroll
            for (int j = 0; j < SUB; ++j) l0 = (uint32_t)ins0(l0, b[j]);
            auto lidx = [&](int r) {
                uint32_t l = l0;
#pragma unroll
                for (int j = 0; j < SUB; ++j) l |= ((r >> j) & 1) ? (1u << b[j]) : 0u;
                return l;
            };
            T v[E];
#pragma unroll
            for (int r = 0; r < E; ++r) v[r] = sm[swz(lidx(r))];
            for (int k = 0; k < nops; ++k) {
                const TileOp &op = ops[rec + k];
                if ((base & op.greq) != op.greq) continue;
                const int sl = op.slot;
                if ((sl & kSlotCtlTest) && !((t >> op.cbit) & 1u)) continue;
                bool t1 = false;
                if (sl & kSlotT1) t1 = op.tbit >= 0 ? ((t >> op.tbit) & 1u) != 0 : (base & op.gtgt) != 0;
                op_dispatch<R, SUB, FMA, CM>(sl & 0xff, v, reinterpret_cast<const R *>(op.u), t1, (sl & kSlotD0) != 0);
            }
            rec += nops;
            // each thread rewrites exactly the slots it read: no barrier before
#pragma unroll
            for (int r = 0; r < E; ++r) sm[swz(lidx(r))] = v[r];
            if (gi == g.ngroups - 1) {
                fence_proxy_async();
                mbar_arrive(bar0 + 8u * (STAGES + s));
            } else {
                cbar();
            }
        }
    }
}

}  // namespace qvg
