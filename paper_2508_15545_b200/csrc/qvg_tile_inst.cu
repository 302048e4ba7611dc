// qvg_tile_inst.cu — the k_tile instantiations of one precision and class
// set (QVG_INST_R, QVG_INST_SET), one object per pair so nvcc compiles them
// in parallel (paper_2508_15545_b200/Makefile).
#include "qvg_tile_select.hpp"

#if !defined(QVG_INST_R) || !defined(QVG_INST_SET)
#error "build with -DQVG_INST_R=double|float -DQVG_INST_SET=0..3"
#endif

#define QVG_CAT3(a, b, c) a##b##_##c
#define QVG_NAME(R, I) QVG_CAT3(tile_kernel_, R, I)

namespace qvg {
TileKernel<QVG_INST_R> QVG_NAME(QVG_INST_R, QVG_INST_SET)(const TileVariant &v) {
    return tile_kernel_pick<QVG_INST_R, kClsSets[QVG_INST_SET]>(v);
}
}  // namespace qvg
