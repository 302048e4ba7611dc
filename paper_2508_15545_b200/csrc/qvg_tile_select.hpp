// qvg_tile_select.hpp — which k_tile instantiation a fused pass launches.
// The instantiations live in separate translation units (qvg_tile_inst.cu,
// compiled once per precision and class set by the Makefile, in parallel);
// the engine gets the kernel's host stub through these functions.
#pragma once

#include "qvg_tile.cuh"
#include "qvg_tile_pipe.cuh"
#include "qvg_tile_ahead.cuh"

namespace qvg {

template <class R>
using TileKernel = void (*)(typename Cplx<R>::T *, const TileParams);

struct TileVariant {
    int sub;     // register subcube bits (3, 4; 5 complex64)
    bool tiny;   // <= 128 threads
    bool small;  // <= 256 threads
    bool fma;    // complex128 DFMA arithmetic (QVG_OPT_FMA)
    bool pf;     // next-tile register prefetch (QVG_OPT_PREFETCH)
    int pipe;    // > 0: k_tile_pipe with this many ring stages (QVG_OPT_PIPE; 128-thread tiles only)
    bool tma;    // k_tile_tma: one tensor-map TMA per tile (QVG_OPT_PIPE 4)
    bool ahead;  // k_tile_ahead: next tile's cp.async load under the last group (QVG_OPT_PIPE 5; 128-thread tiles)
};

// Class-set index: 0 {gen, real, X}, 1 {gen, +-1/2, X}, 2 {gen, +-1/2, sqrt(W)},
// 3 {gen, real u00, X} (qvg_tile.cuh kClsSet*).
constexpr int kClsSets[4] = {kClsSetReal, kClsSetHalf, kClsSetHalfW, kClsSetU3};
inline int class_set_index(int cls_set) {
    return cls_set == kClsSetHalf ? 1 : cls_set == kClsSetHalfW ? 2 : cls_set == kClsSetU3 ? 3 : 0;
}

#define QVG_TILE_SELECT_DECL(R, I) TileKernel<R> tile_kernel_##R##_##I(const TileVariant &v);
QVG_TILE_SELECT_DECL(double, 0)
QVG_TILE_SELECT_DECL(double, 1)
QVG_TILE_SELECT_DECL(double, 2)
QVG_TILE_SELECT_DECL(double, 3)
QVG_TILE_SELECT_DECL(float, 0)
QVG_TILE_SELECT_DECL(float, 1)
QVG_TILE_SELECT_DECL(float, 2)
QVG_TILE_SELECT_DECL(float, 3)
#undef QVG_TILE_SELECT_DECL

template <class R>
inline TileKernel<R> tile_kernel(int set_idx, const TileVariant &v) {
    if constexpr (sizeof(R) == 8) {
        switch (set_idx) {
        case 1: return tile_kernel_double_1(v);
        case 2: return tile_kernel_double_2(v);
        case 3: return tile_kernel_double_3(v);
        default: return tile_kernel_double_0(v);
        }
    } else {
        switch (set_idx) {
        case 1: return tile_kernel_float_1(v);
        case 2: return tile_kernel_float_2(v);
        case 3: return tile_kernel_float_3(v);
        default: return tile_kernel_float_0(v);
        }
    }
}

// The instantiation table for one (precision, class set): included by
// qvg_tile_inst.cu only.
template <class R, int CM>
TileKernel<R> tile_kernel_pick(const TileVariant &v) {
    if (v.ahead && v.small && !v.pf && !v.fma) {  // qvg_tile_ahead.cuh
        if (v.sub == 4) return v.tiny ? k_tile_ahead<R, 4, false, 128, CM> : k_tile_ahead<R, 4, false, 256, CM>;
    }
    if (v.tma && v.tiny && !v.pf) {  // tensor-map pipeline (qvg_tile_pipe.cuh)
        if constexpr (sizeof(R) == 4) {
            if (v.sub == 5) return k_tile_tma<R, 5, false, CM, 2>;
        }
        if (v.sub == 4) return v.fma ? k_tile_tma<R, 4, true, CM, 2> : k_tile_tma<R, 4, false, CM, 2>;
        if (v.sub == 3) return v.fma ? k_tile_tma<R, 3, true, CM, 2> : k_tile_tma<R, 3, false, CM, 2>;
    }
    if (v.pipe > 0 && v.tiny && !v.pf) {  // bulk-copy pipeline (qvg_tile_pipe.cuh)
        if constexpr (sizeof(R) == 4) {
            if (v.sub == 5) return v.pipe >= 3 ? k_tile_pipe<R, 5, false, CM, 3> : k_tile_pipe<R, 5, false, CM, 2>;
        }
        if (v.sub == 4)
            return v.fma ? k_tile_pipe<R, 4, true, CM, 2>
                         : (v.pipe >= 3 ? k_tile_pipe<R, 4, false, CM, 3> : k_tile_pipe<R, 4, false, CM, 2>);
        if (v.sub == 3) return v.fma ? k_tile_pipe<R, 3, true, CM, 2> : k_tile_pipe<R, 3, false, CM, 2>;
    }
    if constexpr (sizeof(R) == 4) {  // 32-amplitude subcubes: complex64 only (64 data registers)
        if (v.sub == 5) return v.tiny ? k_tile<R, 5, false, 128, false, CM> : k_tile<R, 5, false, 256, false, CM>;
    }
    if (v.sub == 4)
        return v.tiny ? (v.fma ? k_tile<R, 4, true, 128, false, CM> : k_tile<R, 4, false, 128, false, CM>)
                      : (v.fma ? k_tile<R, 4, true, 256, false, CM> : k_tile<R, 4, false, 256, false, CM>);
    if (v.pf)
        return v.small ? (v.fma ? k_tile<R, 3, true, 256, true, CM> : k_tile<R, 3, false, 256, true, CM>)
                       : (v.fma ? k_tile<R, 3, true, 512, true, CM> : k_tile<R, 3, false, 512, true, CM>);
    return v.small ? (v.fma ? k_tile<R, 3, true, 256, false, CM> : k_tile<R, 3, false, 256, false, CM>)
                   : (v.fma ? k_tile<R, 3, true, 512, false, CM> : k_tile<R, 3, false, 512, false, CM>);
}

}  // namespace qvg
