// qvg_tile.cuh — K4, the fused tile pass: the B200 replacement for the
// reference's block store + sliding window (reference store.cpp, cache.cpp,
// kernel.cpp:113-146).
//
// A CTA owns a tile of 2^k amplitudes and applies a run of gates to it in
// circuit order, so the whole run costs one HBM round trip instead of one per
// gate. The tile is the set of amplitudes that agree on every qubit outside
// the tile qubit set Q (|Q| = k): its lowest `lowc` qubits are 0..lowc-1
// (contiguous 2^lowc-amplitude segments in HBM, >= 128 B), the other k-lowc
// are arbitrary high qubits, so gates on any qubit can be fused. A control
// outside Q is constant per tile, and a diagonal gate needs no pairing, so its
// qubits may lie anywhere.
//
// Inside the tile the run is cut into groups whose pair ops touch at most SUB
// tile bits. For a group, each of the 2^(k-SUB) threads holds the 2^SUB
// amplitudes of one SUB-bit subcube in registers and applies all the group's
// ops there; shared memory is only the transpose buffer between groups. The
// first group reads HBM directly and the last one writes HBM directly, so a
// run that fits one group never touches the shared tile. The op records (the
// same for every tile) travel in the kernel's parameter bank.
//
// Measured limits (profiles/r01_fused_ab.json, r01_ncu_summary.md): the kernel
// is compute/issue-bound, not HBM-bound — ~52% FP64 pipe, 64% issue slots;
// a bit-exact FP64-instruction reduction for special matrices (real, or with
// exact 0/2^k components) was tried and did not help (reverted), so the next
// lever is latency and per-op overhead, not arithmetic.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "qvg_kernels.cuh"

namespace qvg {

enum TileOpKind : int32_t { TILE_PAIR = 0, TILE_DIAG = 1, TILE_GROUP = 2 };

// One record of a tile pass: a group header followed by its ops.
struct __align__(16) TileOp {
    int32_t kind;      // TileOpKind
    int32_t tbit;      // pair/diag: tile-local target bit (-1: diag target outside Q); group: op count
    int32_t cbit;      // tile-local control bit, -1 if none or outside Q
    int32_t slot;      // pair: index of the target among the group's bits; diag: d0 == 1 exactly
    uint64_t greq;     // global bits that must be 1 in the tile base (controls outside Q)
    uint64_t gtgt;     // diag: global target bit outside Q; group: packed bits b0 | b1<<8 | b2<<16 | b3<<24
    double u[8];       // matrix (diag uses u00 = u[0..1], u11 = u[6..7])
};
static_assert(sizeof(TileOp) == 96, "TileOp layout");

struct TileGeom {
    int n, k, lowc;       // qubits, tile qubits, contiguous low qubits
    int nhi;              // k - lowc
    int ngroups;          // register groups in this pass
    int nrec;             // records (headers + ops)
    int sub;              // subcube bits per thread (3 or 4)
    int pad;
    int hiq[24];          // tile qubits >= lowc, ascending (tile-local bits lowc..k-1)
    uint64_t ntiles;      // 2^(n-k)
};

// Records per fused pass; they travel as the kernel's parameter block
// (CUDA 12.1+ allows 32 KB of parameters).
constexpr int kMaxTileRecs = 256;
struct TileParams {
    TileGeom g;
    TileOp ops[kMaxTileRecs];
};
static_assert(sizeof(TileParams) < 32000, "kernel parameter block limit");

// Shared-tile slot of local index l: the 16-B column within each 128-B row is
// XORed with the row's low bits, so lanes whose amplitudes are 2^3, 2^4 or
// 2^5 apart (a group over the carrier bits) hit different banks.
__device__ __forceinline__ uint32_t swz(uint32_t l) { return l ^ ((l >> 3) & 7u); }

// Pair op over the 2^SUB register amplitudes. Target on register slot J, control on slot K (-1: none / decided per tile):
// both are compile-time, so a controlled op costs exactly its pairs and no
// per-pair tests run (the instruction mix was 60% non-FP64 before this).
template <class R, int SUB, int J, int K, bool FMA>
__device__ __forceinline__ void group_pair(typename Cplx<R>::T (&v)[1 << SUB], const R *u) {
    if constexpr (J < SUB && K < SUB && J != K) {
#pragma unroll
        for (int r = 0; r < (1 << SUB); ++r) {
            if ((r >> J) & 1) continue;
            if (K >= 0 && !((r >> K) & 1)) continue;
            const typename Cplx<R>::T a = v[r], b = v[r | (1 << J)];
            v[r] = madd2x<FMA>(u[0], u[1], a, u[2], u[3], b);
            v[r | (1 << J)] = madd2x<FMA>(u[4], u[5], a, u[6], u[7], b);
        }
    }
}

// slot code = 8*J + (K+1)
template <class R, int SUB, bool FMA>
__device__ __forceinline__ void group_pair_dispatch(int code, typename Cplx<R>::T (&v)[1 << SUB], const R *u) {
#define QVG_GP(J, K) \
    case 8 * (J) + (K) + 1: group_pair<R, SUB, J, K, FMA>(v, u); break;
    switch (code) {
        QVG_GP(0, -1) QVG_GP(0, 1) QVG_GP(0, 2) QVG_GP(0, 3)
        QVG_GP(1, -1) QVG_GP(1, 0) QVG_GP(1, 2) QVG_GP(1, 3)
        QVG_GP(2, -1) QVG_GP(2, 0) QVG_GP(2, 1) QVG_GP(2, 3)
        QVG_GP(3, -1) QVG_GP(3, 0) QVG_GP(3, 1) QVG_GP(3, 2)
    default: break;
    }
#undef QVG_GP
}

// Mask over the subcube: bit r set when element r has tile-local bit `bit`.
template <int SUB>
__device__ __forceinline__ uint32_t sub_mask(int bit, const int (&b)[SUB], uint32_t l0) {
    constexpr uint32_t full = (1u << (1 << SUB)) - 1u;
    if (bit < 0) return full;
    uint32_t m = ((l0 >> bit) & 1u) ? full : 0u;
#pragma unroll
    for (int j = 0; j < SUB; ++j) {
        if (bit == b[j]) {
            uint32_t mj = 0;
#pragma unroll
            for (int r = 0; r < (1 << SUB); ++r) mj |= ((r >> j) & 1) ? (1u << r) : 0u;
            m = mj;
        }
    }
    return m;
}

// MAXT: the largest CTA this instantiation serves (2^(k-SUB) threads). The
// minimum-blocks hint keeps 4 CTAs/SM (64 registers) at 256 threads: measured
// faster than 3 CTAs with 80 registers and no spills (C3 1278 vs 1356 ms).
template <class R, int SUB, bool FMA, int MAXT>
__global__ void __launch_bounds__(MAXT, (MAXT <= 256 && SUB == 3) ? 4 : 2)
k_tile(typename Cplx<R>::T *__restrict__ psi, const __grid_constant__ TileParams prm) {
    using T = typename Cplx<R>::T;
    constexpr int E = 1 << SUB;
    const TileGeom &g = prm.g;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // Op records are read straight from the kernel's parameter (constant)
    // bank: the index is warp-uniform, so they load through the constant
    // cache into uniform registers with no shared-memory traffic.
    const TileOp *ops = prm.ops;
    uint64_t *offhi = reinterpret_cast<uint64_t *>(smem_raw);
    T *sm = reinterpret_cast<T *>(smem_raw + (((sizeof(uint64_t) << g.nhi) + 15) & ~15ull));
    const uint32_t nhi = 1u << g.nhi;
    const uint32_t lowm = (1u << g.lowc) - 1u;
    {  // the high-qubit offset table
        for (uint32_t h = threadIdx.x; h < nhi; h += blockDim.x) {
            uint64_t off = 0;
#pragma unroll
            for (int i = 0; i < 24; ++i)
                if (i < g.nhi && ((h >> i) & 1u)) off |= 1ull << g.hiq[i];
            offhi[h] = off;
        }
    }
    __syncthreads();
    for (uint64_t tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x) {
        // base index: the tile number spread over the qubits outside Q
        uint64_t base = tile << g.lowc;
#pragma unroll
        for (int i = 0; i < 24; ++i)
            if (i < g.nhi) base = ins0(base, g.hiq[i]);
        int rec = 0;
        for (int gi = 0; gi < g.ngroups; ++gi) {
            const int nops = ops[rec].tbit;
            const uint64_t packed = ops[rec].gtgt;
            ++rec;
            int b[SUB];
#pragma unroll
            for (int j = 0; j < SUB; ++j) b[j] = (int)((packed >> (8 * j)) & 0xff);
            // this thread's subcube: local indices l0 | sum_j {0, 2^b_j}
            uint32_t l0 = threadIdx.x;
#pragma unroll
            for (int j = 0; j < SUB; ++j) l0 = (uint32_t)ins0(l0, b[j]);
            auto lidx = [&](int r) {
                uint32_t l = l0;
#pragma unroll
                for (int j = 0; j < SUB; ++j) l |= ((r >> j) & 1) ? (1u << b[j]) : 0u;
                return l;
            };
            T v[E];
            if (gi == 0) {
#pragma unroll
                for (int r = 0; r < E; ++r) {
                    const uint32_t lr = lidx(r);
                    v[r] = ld_amp(psi + (base | offhi[lr >> g.lowc] | (lr & lowm)));
                }
            } else {
#pragma unroll
                for (int r = 0; r < E; ++r) v[r] = sm[swz(lidx(r))];
            }
            // The next op's record is fetched from shared memory while the
            // current one computes (its load latency was the top stall).
            TileOp nxt = ops[rec];
            for (int i = 0; i < nops; ++i) {
                const TileOp op = nxt;
                if (i + 1 < nops) nxt = ops[rec + i + 1];
                if ((base & op.greq) != op.greq) continue;  // control outside the tile is 0
                R u[8];
#pragma unroll
                for (int x = 0; x < 8; ++x) u[x] = (R)op.u[x];
                if (op.kind == TILE_PAIR) {
                    group_pair_dispatch<R, SUB, FMA>(op.slot, v, u);
                } else {
                    const uint32_t cm = sub_mask<SUB>(op.cbit, b, l0);
                    const uint32_t tm = op.tbit >= 0 ? sub_mask<SUB>(op.tbit, b, l0)
                                                     : ((base & op.gtgt) ? 0xFFFFu : 0u);
                    // elements that change: control set and (d0 != 1 or target bit set)
                    const uint32_t sel = cm & (op.slot != 0 ? tm : 0xFFFFu);
#pragma unroll
                    for (int r = 0; r < E; ++r) {
                        if (!((sel >> r) & 1u)) continue;
                        v[r] = ((tm >> r) & 1u) ? cmulx<FMA>(u[6], u[7], v[r]) : cmulx<FMA>(u[0], u[1], v[r]);
                    }
                }
            }
            rec += nops;
            if (gi == g.ngroups - 1) {
#pragma unroll
                for (int r = 0; r < E; ++r) {
                    const uint32_t lr = lidx(r);
                    st_amp(psi + (base | offhi[lr >> g.lowc] | (lr & lowm)), v[r]);
                }
            } else {
#pragma unroll
                for (int r = 0; r < E; ++r) sm[swz(lidx(r))] = v[r];
                __syncthreads();
            }
        }
        if (g.ngroups > 1) __syncthreads();  // last group read sm; the next tile's groups write it
    }
}

}  // namespace qvg
