// qvg_plan.hpp — host-side pass planner (no CUDA calls; unit-testable on CPU
// through qvg_plan_passes).
//
// The reference makes exactly one streaming traversal per gate
// (reference kernel.cpp:132-146: no fusion). The planner maps a
// circuit onto HBM passes instead:
//   * one single-gate pass per op, choosing the kernel that touches the fewest
//     bytes (controlled ops read only control=1 amplitudes, diag(1,d) ops only
//     the amplitudes whose bits are all 1, identities nothing), or
//   * one fused tile pass for a maximal run of consecutive ops whose
//     non-diagonal targets fit in one tile qubit set, when that run would cost
//     more than one full read+write as single passes.
// Ops move only past ops they commute with bit for bit (reorder_for_tiles,
// REORDER_EXACT), so complex128 results stay bit-identical to the reference.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "qvg.h"
#include "qvg_kernels.cuh"
#include "qvg_tile.cuh"

namespace qvg {

struct Validation : std::runtime_error {
    using std::runtime_error::runtime_error;
};

enum PassKind { PASS_PAIRS = 0, PASS_LOW = 1, PASS_PHASE = 2, PASS_TILE = 3, PASS_PERM = 4 };

struct OpInfo {
    bool diag = false;      // u01 == u10 == 0
    bool phase = false;     // diag and u00 == 1 + 0i
    bool identity = false;  // phase and u11 == 1 + 0i
    bool neg = false;       // phase and u11 == -1 + 0i (Z, CZ): a sign flip in fused tiles
    int cls = TILE_CLS_GEN; // non-diagonal: structured-matrix class for fused tiles (qvg_tile.cuh)
    int target = 0;
    int control = -1;
};

// Structured-matrix class of a non-diagonal 2x2 (fused tiles compute these
// with fewer FP64 instructions and the reference's value, qvg_tile.cuh).
inline int pair_class(const double *u) {
    if (u[0] == 0.0 && u[1] == 0.0 && u[2] == 1.0 && u[3] == 0.0 && u[4] == 1.0 && u[5] == 0.0 && u[6] == 0.0 &&
        u[7] == 0.0)
        return TILE_CLS_SWAP;
    if (u[1] == 0.0 && u[3] == 0.0 && u[5] == 0.0 && u[7] == 0.0) return TILE_CLS_REAL;
    auto h = [&](int i) { return u[i] == 0.5 || u[i] == -0.5; };
    bool half = true;
    for (int i = 0; i < 8; ++i) half = half && h(i);
    if (half) return TILE_CLS_HALF;
    if (h(0) && h(1) && h(6) && h(7) && u[2] == 0.0 && u[3] != 0.0 && u[4] != 0.0 && u[5] == 0.0)
        return TILE_CLS_SQW;
    if (u[1] == 0.0) return TILE_CLS_U00R;
    return TILE_CLS_GEN;
}

// The record's u[] for an SQW-class op: (s0/2, -s0 s1, q) for lo (u00 and
// u01 = (0, q)) and (s0'/2, -s0' s1', p) for hi (u11 and u10 = (p, 0)), as
// sqw_lo / sqw_hi (qvg_tile.cuh) expect.
inline void sqw_record(const double *u, double *out) {
    auto sg = [](double x) { return x > 0 ? 1.0 : -1.0; };
    double r[8] = {u[0], -sg(u[0]) * sg(u[1]), u[3], 0.0, u[6], -sg(u[6]) * sg(u[7]), u[4], 0.0};
    std::memcpy(out, r, sizeof(r));
}

// The class set of one fused pass: a k_tile instantiation compiles at most
// three sets of pair bodies without spilling (qvg_tile.cuh), so the pass
// takes the set that saves the most FP64 instructions per pair (real 16,
// X 24, +-1/2 12, sqrt(W) 16, real u00 4); ops of other classes run the
// general body.
inline int tile_class_set(const OpInfo *info, uint64_t begin, uint64_t end) {
    uint64_t n[6] = {};
    for (uint64_t x = begin; x < end; ++x) {
        if (info[x].identity || info[x].diag) continue;
        n[info[x].cls] += 1;
    }
    const uint64_t real = 16 * n[TILE_CLS_REAL] + 24 * n[TILE_CLS_SWAP];
    const uint64_t half = 12 * n[TILE_CLS_HALF] + 24 * n[TILE_CLS_SWAP];
    const uint64_t halfw = 12 * n[TILE_CLS_HALF] + 16 * n[TILE_CLS_SQW];
    const uint64_t u3 = 4 * n[TILE_CLS_U00R] + 24 * n[TILE_CLS_SWAP];
    if (halfw > real && halfw > half && halfw > u3) return kClsSetHalfW;
    if (u3 > real && u3 > half) return kClsSetU3;
    return half > real ? kClsSetHalf : kClsSetReal;
}

// The record's u[] for a HALF-class op: per output row (lo: u00 u01, hi: u10
// u11) the four reals (s0/2, -s0 s1, -s2 s3, s0 s2) that half_apply
// (qvg_tile.cuh) expects, s0..s3 the signs of the row's re/im entries.
inline void half_record(const double *u, double *out) {
    for (int row = 0; row < 2; ++row) {
        const double *m = u + 4 * row;
        const double s0 = m[0] > 0 ? 1.0 : -1.0, s1 = m[1] > 0 ? 1.0 : -1.0;
        const double s2 = m[2] > 0 ? 1.0 : -1.0, s3 = m[3] > 0 ? 1.0 : -1.0;
        out[4 * row + 0] = m[0];
        out[4 * row + 1] = -s0 * s1;
        out[4 * row + 2] = -s2 * s3;
        out[4 * row + 3] = s0 * s2;
    }
}

inline OpInfo classify(const qvg_gate &g) {
    OpInfo o;
    const double *u = g.u;
    o.diag = u[2] == 0.0 && u[3] == 0.0 && u[4] == 0.0 && u[5] == 0.0;
    o.phase = o.diag && u[0] == 1.0 && u[1] == 0.0;
    o.identity = o.phase && u[6] == 1.0 && u[7] == 0.0;
    o.neg = o.phase && u[6] == -1.0 && u[7] == 0.0;
    if (!o.diag) o.cls = pair_class(u);
    o.target = (int)g.target;
    o.control = g.kind == QVG_OP_CONTROLLED ? g.control : -1;
    return o;
}

// Reference validate_circuit (circuit.cpp:31-52) + apply_gate_streamed's
// check (kernel.cpp:134-140).
inline void validate_op(const qvg_gate &g, uint32_t n, uint64_t idx) {
    const std::string at = "op " + std::to_string(idx) + ": ";
    if (g.kind != QVG_OP_SINGLE && g.kind != QVG_OP_CONTROLLED)
        throw Validation(at + "unknown op kind " + std::to_string(g.kind));
    if (g.flags != 0) throw Validation(at + "reserved flags must be 0");
    if (g.target >= n)
        throw Validation(at + "target " + std::to_string(g.target) + " >= n_qubits " + std::to_string(n));
    if (g.kind == QVG_OP_CONTROLLED) {
        if (g.control < 0 || (uint32_t)g.control >= n)
            throw Validation(at + "control " + std::to_string(g.control) + " >= n_qubits " + std::to_string(n));
        if ((uint32_t)g.control == g.target)
            throw Validation(at + "control equals target (" + std::to_string(g.target) + ")");
    }
    for (int i = 0; i < 8; ++i)
        if (!(g.u[i] - g.u[i] == 0.0)) throw Validation(at + "matrix entry is not finite");
}

struct Pass {
    PassKind kind = PASS_PAIRS;
    qvg_gate op{};          // single-gate passes
    OpInfo info{};
    TileGeom geom{};        // tile passes
    uint32_t op_begin = 0;  // into Plan::tile_ops
    uint32_t op_count = 0;
    uint64_t bytes = 0;     // algorithmic HBM bytes (read + write, sector-rounded)
    uint64_t gates = 0;     // circuit ops covered
};

struct Plan {
    std::vector<Pass> passes;
    std::vector<TileOp> tile_ops;
    uint64_t gates = 0;
};

struct PlanOptions {
    uint32_t n = 0;          // qubits addressed by the kernels (local qubits when sharded)
    uint32_t amp_bytes = 16; // 16 complex128, 8 complex64
    bool fuse = true;
    uint32_t tile_qubits = 12;
    uint32_t carriers = 3;
    bool low_kernel = false;
    uint32_t min_run = 32;   // see qvg_state::min_run
    uint32_t sub_bits = 3;   // tile register subcube: 2^sub amplitudes per thread (3..5; 5 complex64 only)
    uint32_t reorder = 2;    // QVG_OPT_REORDER: ReorderMode (below); 2 keeps every bit
    bool classes = true;     // QVG_OPT_CLASSES: structured-matrix op bodies in fused tiles
    uint32_t stage_bits = 3; // stage a first/last group through shared memory when its bits
                             // include tile bits 0..stage_bits-1 (warp lanes >= 2^stage_bits
                             // amplitudes apart); 0 = never
    bool group_reorder = true;  // ops may join an earlier register group of their pass when the reorder rule
                                // allows the move, and an X-class op's control may stay a thread-index bit
    bool perm = false;       // QVG_OPT_PERM: a fused run of only X / CX / Z / CZ ops is a signed
                             // permutation of the tile: one shared-memory scatter (k_tile_perm)
};

// Ops per fused pass: with at most one group header per op the records fit
// the kernel parameter block (kMaxTileRecs).
constexpr uint64_t kMaxRunOps = kMaxTileRecs / 2;

// 2 * touched * S, rounded up to whole 32-B sectors when the touched runs are
// shorter than a sector.
inline uint64_t sector_bytes(uint32_t n, int forced_bits, int lowest_forced, uint32_t S) {
    const uint64_t touched = 1ull << (n - forced_bits);
    uint64_t bytes = 2ull * touched * S;
    if (forced_bits > 0) {
        const uint64_t run = (1ull << lowest_forced) * S;
        if (run < 32) bytes *= 32 / run;
    }
    return std::min<uint64_t>(bytes, 2ull * (1ull << n) * S);
}

inline Pass single_pass(const qvg_gate &g, const OpInfo &o, const PlanOptions &po) {
    Pass p;
    p.op = g;
    p.info = o;
    p.gates = 1;
    const uint32_t n = po.n, S = po.amp_bytes;
    if (o.phase) {
        p.kind = PASS_PHASE;
        const int lowest = o.control >= 0 ? std::min(o.target, o.control) : o.target;
        p.bytes = sector_bytes(n, o.control >= 0 ? 2 : 1, lowest, S);
        return p;
    }
    // Low-target kernel needs 32 consecutive enumerated amplitudes per warp.
    const bool ctl_ins = o.control >= 0 && ((uint64_t)S << o.control) >= po.min_run;
    const uint32_t enum_bits = n - (ctl_ins ? 1 : 0);
    if (po.low_kernel && o.target < 5 && enum_bits >= 5 && n >= 6) {
        p.kind = PASS_LOW;
    } else {
        p.kind = PASS_PAIRS;
    }
    p.bytes = o.control >= 0 ? sector_bytes(n, 1, o.control, S) : 2ull * (1ull << n) * S;
    return p;
}

// FP64 work of a fused pass per amplitude pair, from its records (the op
// bodies of qvg_tile.cuh): general 28, real-u00 24, +-1/2 entries 16, real 12,
// sqrt(W) 12, X 4 (moves through DADD), a phase 6 per multiplied amplitude;
// an op controlled inside its group touches half the pairs. Used to pick the
// kernel per pass (qvg_engine.cu launch_tile): light passes are bound by
// exposed HBM latency, heavy ones by FP64 issue.
inline double tile_pass_weight(const TileOp *recs, int nrec) {
    static const double cls_w[6] = {28, 12, 4, 16, 12, 24};  // TileCls order: GEN REAL SWAP HALF SQW U00R
    double w = 0;
    for (int i = 0; i < nrec; ++i) {
        const TileOp &o = recs[i];
        if (o.kind == TILE_GROUP) continue;
        const int d = o.slot & 0xff;
        if (d < kDispDiag) {
            const int cls = d / 30, k = (d % 30) % 6;  // k = K + 1: 0 = no control in the group
            w += cls_w[cls < 6 ? cls : 0] * (k || (o.slot & kSlotCtlTest) ? 0.5 : 1.0);
        } else {
            const int dd = d - kDispDiag;
            if (dd >= 36) continue;  // sign flips: no FP64
            const int j = dd / 6, k = dd % 6;  // j = J + 1 (0: target outside the group), k = K + 1
            double x = j ? 6.0 : 12.0 * 0.5;   // target in the group: half the amplitudes; else t1 decides (half the threads)
            if (o.slot & kSlotD0) x *= 2;
            if (k) x *= 0.5;
            if (o.slot & kSlotCtlTest) x *= 0.5;
            w += x;
        }
    }
    return w;
}

// Global index offset of tile-local bit p: the low carriers map to
// themselves, bits >= lowc to their high qubits.
inline uint64_t tile_bit_offset(const TileGeom &g, int p) {
    return p < g.lowc ? 1ull << p : 1ull << g.hiq[p - g.lowc];
}

inline int local_bit(int q, const TileGeom &g) {
    if (q < g.lowc) return q;
    for (int i = 0; i < g.nhi; ++i)
        if (g.hiq[i] == q) return g.lowc + i;
    return -1;
}

// Commutation-aware op order for fusion (QVG_OPT_REORDER). The tile runs are
// built greedily as in make_plan, but an op that does not fit the current run
// no longer ends it. Its qubits are marked blocked, and later ops that touch
// no blocked qubit join the run: such an op acts on qubits disjoint from every
// op it overtakes, so the two commute.
//   REORDER_ANY (1): any such move. The product is mathematically the same,
//     but amplitudes see the products in another order, so results differ
//     from the reference in the last bits (tests bound them at 1e-12).
//   REORDER_EXACT (2, default): only moves that keep every bit. A permutation
//     (X, CX: the amplitudes move, no arithmetic) or a +-1 phase (Z, CZ: an
//     exact negation, which commutes with round-to-nearest) on disjoint
//     qubits commutes bit for bit with any op, so a move is allowed when the
//     moved op or every op it overtakes is one of these. Two general ops are
//     never swapped.
enum ReorderMode : uint32_t { REORDER_NONE = 0, REORDER_ANY = 1, REORDER_EXACT = 2 };

inline bool exact_commuter(const OpInfo &o) {
    return o.identity || o.neg || (!o.diag && o.cls == TILE_CLS_SWAP);
}

// `order`, if given, receives the source index of each output op.
inline std::vector<qvg_gate> reorder_for_tiles(const qvg_gate *ops, uint64_t count, const PlanOptions &po,
                                               std::vector<uint64_t> *order = nullptr) {
    constexpr uint64_t kWindow = 512;  // look-ahead per run
    const uint32_t n = po.n;
    const uint32_t k = std::min<uint32_t>(po.tile_qubits, n);
    const uint32_t lowmin = std::min<uint32_t>(po.carriers, k);
    std::vector<qvg_gate> out;
    out.reserve(count);
    std::vector<char> taken(count, 0);
    uint64_t first = 0;  // lowest index not yet emitted
    while (first < count) {
        std::vector<int> high;
        std::vector<char> blocked(n, 0);
        bool general_skipped = false;  // a skipped op that is not an exact commuter
        uint64_t live = 0;
        for (uint64_t j = first; j < count && j < first + kWindow && live < kMaxRunOps; ++j) {
            if (taken[j]) continue;
            const qvg_gate &g = ops[j];
            const OpInfo o = classify(g);
            const bool blk = blocked[o.target] || (o.control >= 0 && blocked[o.control]);
            bool fits = !blk;
            if (fits && po.reorder == REORDER_EXACT && general_skipped && !exact_commuter(o)) fits = false;
            if (fits && !o.identity && !o.diag && (uint32_t)o.target >= lowmin &&
                std::find(high.begin(), high.end(), o.target) == high.end()) {
                if (high.size() == k - lowmin) fits = false;
                else high.push_back(o.target);
            }
            if (!fits) {
                blocked[o.target] = 1;
                if (o.control >= 0) blocked[o.control] = 1;
                general_skipped = general_skipped || !exact_commuter(o);
                continue;
            }
            taken[j] = 1;
            out.push_back(g);
            if (order) order->push_back(j);
            live += o.identity ? 0 : 1;
        }
        while (first < count && taken[first]) ++first;
    }
    return out;
}

inline Plan make_plan(const qvg_gate *ops, uint64_t count, const PlanOptions &po) {
    Plan plan;
    const uint32_t n = po.n;
    const uint64_t full = 2ull * (1ull << n) * po.amp_bytes;
    const uint32_t k = std::min<uint32_t>(po.tile_qubits, n);
    const bool fuse = po.fuse && k >= 5;  // a tile needs >= 4 threads of 8-amplitude subcubes
    const uint32_t lowmin = std::min<uint32_t>(po.carriers, k);
    const uint32_t sub = po.sub_bits;
    std::vector<OpInfo> info(count);
    for (uint64_t i = 0; i < count; ++i) info[i] = classify(ops[i]);
    plan.gates = count;

    uint64_t i = 0;
    while (i < count) {
        if (!fuse) {
            if (!info[i].identity) plan.passes.push_back(single_pass(ops[i], info[i], po));
            ++i;
            continue;
        }
        // Greedy maximal run whose non-diagonal targets fit in one tile.
        std::vector<int> high;  // tile qubits >= lowmin required by the run
        uint64_t j = i, cost = 0, live = 0;
        while (j < count && live < kMaxRunOps) {
            const OpInfo &o = info[j];
            if (!o.identity) {
                if (!o.diag && (uint32_t)o.target >= lowmin &&
                    std::find(high.begin(), high.end(), o.target) == high.end()) {
                    if (high.size() == k - lowmin) break;
                    high.push_back(o.target);
                }
                cost += single_pass(ops[j], o, po).bytes;
                ++live;
            }
            ++j;
        }
        if (j == i) {  // degenerate tile geometry: nothing fits, fall back
            plan.passes.push_back(single_pass(ops[i], info[i], po));
            ++i;
            continue;
        }
        if (live >= 2 && cost > full) {
            // Tile qubit set Q: carriers 0..lowmin-1, the run's high targets,
            // then the lowest free qubits until |Q| = k.
            std::vector<char> inq(n, 0);
            for (uint32_t q = 0; q < lowmin; ++q) inq[q] = 1;
            for (int q : high) inq[q] = 1;
            uint32_t size = lowmin + (uint32_t)high.size();
            for (uint32_t q = 0; q < n && size < k; ++q)
                if (!inq[q]) { inq[q] = 1; ++size; }
            TileGeom g{};
            g.n = (int)n;
            g.k = (int)k;
            g.lowc = 0;
            while (g.lowc < (int)n && inq[g.lowc]) ++g.lowc;
            g.nhi = 0;
            for (uint32_t q = (uint32_t)g.lowc; q < n; ++q)
                if (inq[q]) g.hiq[g.nhi++] = (int)q;
            g.ntiles = 1ull << (n - k);
            g.sub = (int)std::min<uint32_t>(sub, k - 2);
            for (int s = 0; s < g.sub; ++s) g.sdep[s] = tile_bit_offset(g, g.k - g.sub + s);
            Pass p;
            p.kind = PASS_TILE;
            p.op_begin = (uint32_t)plan.tile_ops.size();
            // Records: [group header, its ops]... Each group's pair ops touch
            // at most `sub` tile bits (the thread's register subcube).
            std::vector<TileOp> group;
            uint32_t first_low = 0, last_low = 0;  // see PlanOptions::stage_bits
            int gbits[5];
            int nb = 0;
            auto close_group = [&] {
                if (group.empty()) return;
                auto used = [&](int b) {
                    for (int x = 0; x < nb; ++x)
                        if (gbits[x] == b) return true;
                    return false;
                };
                // Pad the free slots with the tile bits the group's diagonal
                // ops use most (their multiplies then skip the elements the
                // bit excludes at compile time).
                int freq[64] = {};
                for (const TileOp &t : group) {
                    if (t.kind != TILE_DIAG) continue;
                    if (t.tbit >= 0) freq[t.tbit] += 2;  // a target halves d0 == 1 work
                    if (t.cbit >= 0) freq[t.cbit] += 1;
                }
                while (nb < g.sub) {
                    int best = -1;
                    for (int b = 0; b < g.k; ++b)
                        if (freq[b] > 0 && !used(b) && (best < 0 || freq[b] > freq[best])) best = b;
                    if (best < 0) break;
                    gbits[nb++] = best;
                }
                // Remaining slots take the HIGHEST unused tile bits: the
                // lanes of a warp then run over the lowest tile bits, so the
                // first group's HBM loads and the last group's stores are
                // contiguous 512-B warp accesses and the shared-memory
                // transposes stay conflict-free.
                for (int b = g.k - 1; nb < g.sub && b >= 0; --b)
                    if (!used(b)) gbits[nb++] = b;
                std::sort(gbits, gbits + g.sub);
                for (TileOp &t : group) {
                    // slot = dispatch index | flags (op_dispatch, qvg_tile.cuh), J / K the
                    // target / control register slots (-1: not in the group). Before this
                    // point slot holds the class (pair) or the d0 == 1 / neg flags (diag,
                    // bits 0 / 1).
                    int J = -1, K = -1;
                    for (int s = 0; s < g.sub; ++s) {
                        if (t.tbit >= 0 && gbits[s] == t.tbit) J = s;
                        if (t.cbit >= 0 && gbits[s] == t.cbit) K = s;
                    }
                    auto tpos = [&](int p) {  // thread-index bit of a tile bit outside the group
                        int below = 0;
                        for (int x = 0; x < g.sub; ++x) below += gbits[x] < p;
                        return p - below;
                    };
                    if (t.kind == TILE_PAIR) {
                        t.slot = 30 * t.slot + 6 * J + K + 1;
                        if (K < 0 && t.cbit >= 0) {  // an X-class op's control left outside the group: tested per thread
                            t.slot |= kSlotCtlTest;
                            t.cbit = tpos(t.cbit);
                        }
                    } else {
                        const bool neg = (t.slot & 2) != 0, d0one = (t.slot & 1) != 0;
                        t.slot = kDispDiag + (neg ? 36 : 0) + 6 * (J + 1) + K + 1;
                        if (K < 0 && t.cbit >= 0) t.slot |= kSlotCtlTest;
                        if (J < 0) t.slot |= kSlotT1;
                        if (!neg && !d0one) t.slot |= kSlotD0;
                        // A tile bit outside the group is a bit of the thread index:
                        // store that position, so the kernel tests threadIdx.x (which
                        // it can re-read) instead of the subcube base l0 (which it
                        // spilled under the 96-register limit and reloaded per op).
                        if (K < 0 && t.cbit >= 0) t.cbit = tpos(t.cbit);
                        if (J < 0 && t.tbit >= 0) t.tbit = tpos(t.tbit);
                    }
                }
                TileOp h{};
                h.kind = TILE_GROUP;
                h.tbit = (int32_t)group.size();
                for (int s = 0; s < g.sub; ++s) h.gtgt |= (uint64_t)gbits[s] << (8 * s);
                for (int s = 0; s < g.sub; ++s) {  // global offsets of the group's bits
                    const uint64_t d = tile_bit_offset(g, gbits[s]);
                    std::memcpy(&h.u[s], &d, sizeof(d));
                }
                uint32_t low = 0;  // lowest tile bits the group holds: its lanes are 2^low amplitudes apart
                while ((int)low < g.sub && gbits[low] == (int)low) ++low;
                if (g.ngroups == 0) first_low = low;
                last_low = low;
                plan.tile_ops.push_back(h);
                plan.tile_ops.insert(plan.tile_ops.end(), group.begin(), group.end());
                group.clear();
                nb = 0;
                g.ngroups += 1;
            };
            // A run of only permutations and +-1 phases (X, CX, SWAP's CXs, Z,
            // CZ) moves each amplitude, changing at most its sign: k_tile_perm
            // applies it as one scatter through shared memory (records: the
            // tile-local target / control bits in op order, qvg_tile_perm.cuh).
            bool perm = po.perm && po.classes;
            for (uint64_t x = i; x < j && perm; ++x) {
                const OpInfo &o = info[x];
                perm = o.identity || o.neg || (!o.diag && o.cls == TILE_CLS_SWAP);
            }
            if (perm) {
                g.ngroups = 0;
                g.stage = 0;
                g.cls_set = 0;
                for (uint64_t x = i; x < j; ++x) {
                    const OpInfo &o = info[x];
                    if (o.identity) continue;
                    TileOp t{};
                    t.kind = o.diag ? TILE_DIAG : TILE_PAIR;
                    t.tbit = local_bit(o.target, g);
                    if (t.tbit < 0) t.gtgt = 1ull << o.target;  // a sign flip decided per tile
                    t.cbit = -1;
                    if (o.control >= 0) {
                        t.cbit = local_bit(o.control, g);
                        if (t.cbit < 0) t.greq = 1ull << o.control;
                    }
                    plan.tile_ops.push_back(t);
                }
                g.nrec = (int)(plan.tile_ops.size() - p.op_begin);
                p.kind = PASS_PERM;
                p.geom = g;
                p.op_count = (uint32_t)g.nrec;
                p.bytes = full;
                p.gates = j - i;
                plan.passes.push_back(p);
                i = j;
                continue;
            }
            g.ngroups = 0;
            g.cls_set = po.classes ? tile_class_set(info.data(), i, j) : (1 << TILE_CLS_GEN);
            // Ops join register groups in circuit order, except that (QVG_OPT_REORDER
            // on) an op further down the run may join the CURRENT group when it fits
            // the group's bits and may move ahead of every op skipped so far: disjoint
            // qubits, and with REORDER_EXACT the moved op is an exact commuter
            // (permutation or sign flip) unless only such ops were skipped (the rule of
            // reorder_for_tiles). A U3 layer followed by a CX ladder then needs one
            // group per 4 qubits instead of one for the layer and one per 3 CX.
            std::vector<uint64_t> pend;
            for (uint64_t x = i; x < j; ++x)
                if (!info[x].identity) pend.push_back(x);
            std::vector<char> done(pend.size(), 0);
            std::vector<char> blocked(n, 0);
            size_t first = 0;
            while (first < pend.size()) {
                std::fill(blocked.begin(), blocked.end(), 0);
                bool general_skipped = false, any_skipped = false;
                for (size_t q = first; q < pend.size(); ++q) {
                    if (done[q]) continue;
                    const uint64_t x = pend[q];
                    const OpInfo &o = info[x];
                    bool ok = !(blocked[o.target] || (o.control >= 0 && blocked[o.control]));
                    if (ok && any_skipped && (po.reorder == REORDER_NONE || !po.group_reorder)) ok = false;
                    if (ok && po.reorder == REORDER_EXACT && general_skipped && !exact_commuter(o)) ok = false;
                    TileOp t{};
                    int need[2] = {-1, -1};
                    if (ok) {
                        std::memcpy(t.u, ops[x].u, sizeof(t.u));
                        t.kind = o.diag ? TILE_DIAG : TILE_PAIR;
                        t.tbit = local_bit(o.target, g);
                        if (t.tbit < 0) t.gtgt = 1ull << o.target;
                        t.cbit = -1;
                        if (o.control >= 0) {
                            t.cbit = local_bit(o.control, g);
                            if (t.cbit < 0) t.greq = 1ull << o.control;
                        }
                        if (t.kind == TILE_DIAG)  // d0 == 1 / neg flags, coded in close_group
                            t.slot = (ops[x].u[0] == 1.0 && ops[x].u[1] == 0.0 ? 1 : 0) | (po.classes && o.neg ? 2 : 0);
                        else
                            t.slot = ((g.cls_set >> o.cls) & 1) ? o.cls : TILE_CLS_GEN;
                        if (t.kind == TILE_PAIR) {
                            // The target must be a register bit. An in-tile control is
                            // made one too: the control test is then the same for every
                            // thread (no lane divergence) and skips half the pairs. An
                            // X-class op (CX: its body only moves amplitudes) whose
                            // control does not fit the group keeps it as a bit of the
                            // thread index instead (tested per thread, like a diagonal
                            // op's control): threads with control 0 skip the op.
                            need[0] = t.tbit;
                            need[1] = t.cbit;
                            auto missing = [&] {
                                int m = 0;
                                for (int y : need) {
                                    if (y < 0) continue;
                                    bool have = false;
                                    for (int bb = 0; bb < nb; ++bb) have |= gbits[bb] == y;
                                    m += have ? 0 : 1;
                                }
                                return m;
                            };
                            if (nb + missing() > (int)g.sub && t.slot == TILE_CLS_SWAP && t.cbit >= 0 && po.group_reorder)
                                need[1] = -1;
                            if (nb + missing() > (int)g.sub) ok = false;  // not this group's (a fresh group always fits)
                        }
                    }
                    if (!ok) {
                        blocked[o.target] = 1;
                        if (o.control >= 0) blocked[o.control] = 1;
                        general_skipped = general_skipped || !exact_commuter(o);
                        any_skipped = true;
                        continue;
                    }
                    if (t.kind == TILE_PAIR && t.slot == TILE_CLS_HALF) half_record(ops[x].u, t.u);
                    if (t.kind == TILE_PAIR && t.slot == TILE_CLS_SQW) sqw_record(ops[x].u, t.u);
                    if (po.amp_bytes == 8) {  // complex64: the kernel reads 8 floats (no F2F per use)
                        float f[8];
                        for (int e = 0; e < 8; ++e) f[e] = (float)t.u[e];
                        std::memset(t.u, 0, sizeof(t.u));
                        std::memcpy(t.u, f, sizeof(f));
                    }
                    for (int y : need) {
                        if (y < 0) continue;
                        bool have = false;
                        for (int bb = 0; bb < nb; ++bb) have |= gbits[bb] == y;
                        if (!have) gbits[nb++] = y;
                    }
                    group.push_back(t);
                    done[q] = 1;
                }
                close_group();
                while (first < pend.size() && done[first]) ++first;
            }
            g.stage = 0;
            if (po.stage_bits > 0) {
                if (first_low >= po.stage_bits) g.stage |= 1;
                if (last_low >= po.stage_bits) g.stage |= 2;
            }
            g.nrec = (int)(plan.tile_ops.size() - p.op_begin);
            p.geom = g;
            p.op_count = (uint32_t)(plan.tile_ops.size() - p.op_begin);
            p.bytes = full;
            p.gates = j - i;
            plan.passes.push_back(p);
        } else {
            for (uint64_t x = i; x < j; ++x)
                if (!info[x].identity) plan.passes.push_back(single_pass(ops[x], info[x], po));
        }
        i = j;
    }
    return plan;
}

// The plan qvg_apply runs for a list of local ops: with REORDER_EXACT the
// bit-exact reordering is kept only when it saves passes (it moves sign flips
// and permutations, which can also scatter a pass's op bodies without saving
// a pass: config 3 measured 3% slower); REORDER_ANY always reorders.
inline Plan plan_ops(const qvg_gate *ops, uint64_t count, const PlanOptions &po) {
    if (!po.reorder || !po.fuse || std::min(po.tile_qubits, po.n) < 5) return make_plan(ops, count, po);
    const std::vector<qvg_gate> moved = reorder_for_tiles(ops, count, po);
    Plan a = make_plan(moved.data(), count, po);
    if (po.reorder == REORDER_ANY) return a;
    Plan b = make_plan(ops, count, po);
    return a.passes.size() < b.passes.size() ? a : b;
}

}  // namespace qvg
