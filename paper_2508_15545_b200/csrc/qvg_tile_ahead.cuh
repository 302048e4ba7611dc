// qvg_tile_ahead.cuh — K4c, the fused tile pass with the NEXT tile's HBM load
// in flight under the current tile's last register group, at k_tile's
// occupancy (no second buffer, no registers held by loads in flight).
//
// tools/tile_trace.py (phase stamps of k_tile, profiles/r02_tile_trace.json)
// shows why k_tile runs below both of its rooflines: a CTA's load, register
// groups and stores are serial, each latency-bound, and with 5 CTAs of 4 warps
// per SM (96 registers per thread) a tile's load is in flight for only ~15% of
// its CTA's time, so an SM keeps about one tile of bytes in flight where the
// HBM rate needs 2.5. The access pattern itself streams at 0.9-1.0 of HBM from
// the same 5 CTAs per SM (tools/native/tile_pattern.cu).
//
// The shared tile buffer is idle from the moment the last group has read it
// into registers until the next tile's first group writes it. This kernel
// fills that window: a CTA runs several tiles; after the last group's reads
// (one barrier) every thread issues the next tile's amplitudes as 16-byte
// cp.async copies (LDGSTS, global -> shared, no registers) into the SAME
// buffer, in k_tile's staged layout (local index t + j * blockDim at
// swz(index)). They land while the last group's ops run and its stores drain,
// so the next tile's first group reads shared memory like every other group.
// A last group that must leave through the buffer (stage bit 1: it holds
// the lowest tile bits) issues the copies after its stores instead.
//
// Same records, op bodies (TileOpsRuntime) and arithmetic as k_tile:
// bit-identical results. complex128 and complex64 (16-amplitude subcubes).
#pragma once

#include "qvg_tile.cuh"

namespace qvg {

template <int BYTES>
__device__ __forceinline__ void cp_async_amp(void *smem_dst, const void *gmem_src) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// (6 CTAs per SM instead of 5, i.e. 80 registers: spills; QFT -7%, ladder +15%, not kept.
// Requesting the next record's dispatch word before an op's body: C3 +1.5%, not kept.)
template <class R, int SUB, bool FMA, int MAXT, int CM>
__global__ void __launch_bounds__(MAXT, (tile_min_blocks<R, SUB, MAXT, false>()))
k_tile_ahead(typename Cplx<R>::T *__restrict__ psi, const __grid_constant__ TileParams prm) {
    using T = typename Cplx<R>::T;
    constexpr int E = 1 << SUB;
    const TileGeom &g = prm.g;
    TileTrace trc;
    trc.enter();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const TileOp *ops = prm.ops;
    uint64_t *offhi = reinterpret_cast<uint64_t *>(smem_raw);
    T *sm = reinterpret_cast<T *>(smem_raw + (((sizeof(uint64_t) << g.nhi) + 15) & ~15ull));
    const uint32_t nhi = 1u << g.nhi;
    const uint32_t lowm = (1u << g.lowc) - 1u;
    for (uint32_t h = threadIdx.x; h < nhi; h += blockDim.x) {
        uint64_t off = 0;
        for (int i = 0; i < g.nhi; ++i)
            if ((h >> i) & 1u) off |= 1ull << g.hiq[i];
        offhi[h] = off;
    }
    __syncthreads();
    auto tile_base = [&](uint64_t tile) {
        uint64_t base = tile << g.lowc;
        for (int i = 0; i < g.nhi; ++i) base = ins0(base, g.hiq[i]);
        return base;
    };
    // the tile's amplitudes, coalesced (lane = consecutive amplitudes), into the swizzled buffer
    // (addresses as in k_tile's staged path: one offset-table lookup per thread,
    // then the planner's offsets of the index bits above the thread index;
    // swz(t + j * blockDim) = swz(t) + j * blockDim for 128-thread CTAs)
    const uint32_t st = swz(threadIdx.x);
    auto fetch = [&](uint64_t tb) {
        const uint64_t dt = tb | offhi[threadIdx.x >> g.lowc] | (threadIdx.x & lowm);
#pragma unroll 4
        for (int j = 0; j < E; ++j) {
            uint64_t a = dt;
#pragma unroll
            for (int i = 0; i < SUB; ++i)
                if ((j >> i) & 1) a |= g.sdep[i];
            cp_async_amp<(int)sizeof(T)>(sm + st + (uint32_t)j * MAXT, psi + a);
        }
        cp_async_commit();
    };
    const TileRange tr = tile_range(g);
    if (tr.first < tr.end) fetch(tile_base(tr.first));
    for (uint64_t tile = tr.first; tile < tr.end; tile += tr.step) {
        const uint64_t base = tile_base(tile);
        const bool more = tile + tr.step < tr.end;
        trc.begin(g, tile);
        cp_async_wait_all();
        __syncthreads();  // every thread's copies have landed
        trc.mark(21);
        int rec = 0;
        for (int gi = 0; gi < g.ngroups; ++gi) {
            const int nops = ops[rec].tbit;
            const uint64_t packed = ops[rec].gtgt;
            // global offsets of the group's bits (the planner's group header, as in k_tile)
            const uint64_t *gdep = reinterpret_cast<const uint64_t *>(ops[rec].u);
            ++rec;
            int b[SUB];
#pragma unroll
            for (int j = 0; j < SUB; ++j) b[j] = (int)((packed >> (8 * j)) & 0xff);
            uint32_t l0 = threadIdx.x;
#pragma unroll
            for (int j = 0; j < SUB; ++j) l0 = (uint32_t)ins0(l0, b[j]);
            // Shared slot of subcube amplitude r: swz is XOR-linear and l0 has
            // zeros at the group's bits, so swz(l0 | bits(r)) = swz(l0) ^ XOR_j
            // r_j swz(2^b_j): one XOR per slot instead of ORs, a shift and a mask.
            uint32_t s0, sb[SUB];
            auto slots = [&]() {
                s0 = swz(l0);
#pragma unroll
                for (int j = 0; j < SUB; ++j) sb[j] = swz(1u << b[j]);
            };
            auto sidx = [&](int r) {
                uint32_t x = s0;
#pragma unroll
                for (int j = 0; j < SUB; ++j) x ^= ((r >> j) & 1) ? sb[j] : 0u;
                return x;
            };
            const bool last = gi == g.ngroups - 1;
            T v[E];
            slots();
#pragma unroll
            for (int r = 0; r < E; ++r) v[r] = sm[sidx(r)];
            if (last && !(g.stage & 2)) {
                __syncthreads();  // the buffer has been read by everyone: refill it under this group's ops
                if (more) fetch(tile_base(tile + tr.step));
            }
            trc.mark_after(6 + 3 * gi, v[0].x, v[E - 1].y);
            TileOpsRuntime::template apply<R, SUB, FMA, CM>(gi, v, base, ops, rec, nops);
            rec += nops;
            trc.mark_after(7 + 3 * gi, v[0].x, v[E - 1].y);
            // the slot indices and addresses are recomputed after the op loop
            // (the asm hides the equality): kept live across it they spill
            asm volatile("" : "+r"(l0));
#pragma unroll
            for (int j = 0; j < SUB; ++j) asm volatile("" : "+r"(b[j]));
            if (!last) {
                // each thread rewrites exactly the slots it read
                slots();
#pragma unroll
                for (int r = 0; r < E; ++r) sm[sidx(r)] = v[r];
                __syncthreads();
            } else if (g.stage & 2) {
                slots();
#pragma unroll
                for (int r = 0; r < E; ++r) sm[sidx(r)] = v[r];
                __syncthreads();
#pragma unroll
                for (int j = 0; j < E; ++j) v[j] = sm[st + (uint32_t)j * MAXT];
                const uint64_t dt = base | offhi[threadIdx.x >> g.lowc] | (threadIdx.x & lowm);
#pragma unroll
                for (int j = 0; j < E; ++j) {
                    uint64_t a = dt;
#pragma unroll
                    for (int i = 0; i < SUB; ++i)
                        if ((j >> i) & 1) a |= g.sdep[i];
                    st_amp(psi + a, v[j]);
                }
                __syncthreads();
                if (more) fetch(tile_base(tile + tr.step));
            } else {
                // amplitude r of the subcube sits at base | dep(l0) | OR_j r_j gdep[j]
                const uint64_t dl0 = base | offhi[l0 >> g.lowc] | (l0 & lowm);
#pragma unroll
                for (int r = 0; r < E; ++r) {
                    uint64_t a = dl0;
#pragma unroll
                    for (int j = 0; j < SUB; ++j)
                        if ((r >> j) & 1) a |= gdep[j];
                    st_amp(psi + a, v[r]);
                }
            }
            trc.mark(8 + 3 * gi);
        }
        trc.end(g.ngroups);
    }
}

}  // namespace qvg
