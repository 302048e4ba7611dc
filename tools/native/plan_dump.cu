// plan_dump.cu — print the fused-pass plan qvg_apply builds for an op list
// (host-only; qvg_plan.hpp). Input: raw qvg_gate records (circuit.gates()).
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include -I paper_2508_15545_b200/csrc tools/native/plan_dump.cu -o /tmp/plan_dump
//     (+ paper_2508_15545_b200/csrc/qvg_jit.cu -I paper_2508_15545_b200/build -ldl for the JIT source)
//   /tmp/plan_dump ops.bin n [tile_qubits=11] [sub=4] [amp_bytes=16] [verbose=0] [jit_pass=-1]
// jit_pass >= 0: print that fused pass's JIT-specialised source (qvg_jit.hpp) instead.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "qvg_jit.hpp"
#include "qvg_plan.hpp"

using namespace qvg;

int main(int argc, char **argv) {
    if (argc < 3) return 2;
    FILE *f = std::fopen(argv[1], "rb");
    if (!f) return 2;
    std::vector<qvg_gate> ops;
    qvg_gate g;
    while (std::fread(&g, sizeof g, 1, f) == 1) ops.push_back(g);
    std::fclose(f);
    PlanOptions po;
    po.n = (uint32_t)std::atoi(argv[2]);
    po.tile_qubits = argc > 3 ? (uint32_t)std::atoi(argv[3]) : 11;
    po.sub_bits = argc > 4 ? (uint32_t)std::atoi(argv[4]) : 4;
    po.amp_bytes = argc > 5 ? (uint32_t)std::atoi(argv[5]) : 16;
    const int verbose = argc > 6 ? std::atoi(argv[6]) : 0;
    const Plan plan = plan_ops(ops.data(), ops.size(), po);
    const int jit_pass = argc > 7 ? std::atoi(argv[7]) : -1;
    if (jit_pass >= 0 && jit_pass < (int)plan.passes.size() && plan.passes[jit_pass].kind == PASS_TILE) {
        const Pass &p = plan.passes[jit_pass];
        const int threads = 1 << (p.geom.k - p.geom.sub);
        const JitVariant v{(int)po.amp_bytes, p.geom.sub, false, threads <= 128 ? 128 : threads <= 256 ? 256 : 512,
                           p.geom.cls_set == kClsSetHalf    ? kClsSetHalf
                           : p.geom.cls_set == kClsSetHalfW ? kClsSetHalfW
                           : p.geom.cls_set == kClsSetU3    ? kClsSetU3
                                                            : kClsSetReal};
        std::fputs(jit_source(p.geom, plan.tile_ops.data() + p.op_begin, v).c_str(), stdout);
        return 0;
    }
    std::printf("ops %zu passes %zu\n", ops.size(), plan.passes.size());
    int pi = 0;
    for (const Pass &p : plan.passes) {
        if (p.kind != PASS_TILE) {
            std::printf("pass %d single kind %d target %d control %d\n", pi++, (int)p.kind, p.op.target, p.op.control);
            continue;
        }
        const TileGeom &gm = p.geom;
        std::printf("pass %d tile gates %llu groups %d recs %d lowc %d stage %d cls %d weight %.0f hiq", pi++,
                    (unsigned long long)p.gates, gm.ngroups, gm.nrec, gm.lowc, gm.stage, gm.cls_set,
                    tile_pass_weight(plan.tile_ops.data() + p.op_begin, gm.nrec));
        for (int i = 0; i < gm.nhi; ++i) std::printf(" %d", gm.hiq[i]);
        std::printf("\n");
        int rec = 0;
        for (int gi = 0; gi < gm.ngroups; ++gi) {
            const TileOp &h = plan.tile_ops[p.op_begin + rec];
            const int nops = h.tbit;
            int npair = 0, ndiag = 0, ctest = 0, t1 = 0, d0 = 0, skipg = 0;
            for (int i = 0; i < nops; ++i) {
                const TileOp &o = plan.tile_ops[p.op_begin + rec + 1 + i];
                if (o.kind == TILE_PAIR) ++npair;
                else {
                    ++ndiag;
                    ctest += (o.slot & kSlotCtlTest) != 0;
                    t1 += (o.slot & kSlotT1) != 0 && o.tbit >= 0;
                    skipg += (o.slot & kSlotT1) != 0 && o.tbit < 0;
                    d0 += (o.slot & kSlotD0) != 0;
                }
            }
            std::printf("  group %d bits", gi);
            for (int s = 0; s < gm.sub; ++s) std::printf(" %d", (int)((h.gtgt >> (8 * s)) & 0xff));
            std::printf(" | ops %d pair %d diag %d (ctl-thread-test %d, tgt-thread %d, tgt-global %d, d0 %d)\n", nops,
                        npair, ndiag, ctest, t1, skipg, d0);
            if (verbose)
                for (int i = 0; i < nops; ++i) {
                    const TileOp &o = plan.tile_ops[p.op_begin + rec + 1 + i];
                    std::printf("    %s slot %d tbit %d cbit %d greq %llx\n", o.kind == TILE_PAIR ? "pair" : "diag",
                                o.slot & 0xff, o.tbit, o.cbit, (unsigned long long)o.greq);
                }
            rec += 1 + nops;
        }
    }
    return 0;
}
