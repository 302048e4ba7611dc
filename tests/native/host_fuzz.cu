// host_fuzz.cu — sanitizer harness for the host-side planning logic (no GPU
// needed). Built with nvcc and -fsanitize=address,undefined by
// tests/test_native_sanitizers.py. It drives:
//   * make_plan / reorder_for_tiles (qvg_plan.hpp);
//   * schedule_ops / schedule_canonicalize (qvg_schedule.hpp);
// over random op lists, options and shard counts, and checks their
// invariants. The reference has no sanitizer coverage (SURVEY §5:
// "-Wall -Wextra" only); this is the B200 build's host-side equivalent of
// compute-sanitizer on the kernels.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "qvg_plan.hpp"
#include "qvg_schedule.hpp"

using namespace qvg;

static int failures = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        if (!(c)) {                                                           \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                                       \
        }                                                                     \
    } while (0)

static qvg_gate random_gate(std::mt19937_64 &rng, uint32_t n) {
    qvg_gate g{};
    std::uniform_int_distribution<uint32_t> q(0, n - 1);
    g.target = q(rng);
    g.control = -1;
    g.kind = QVG_OP_SINGLE;
    if (n >= 2 && rng() % 3 == 0) {
        g.kind = QVG_OP_CONTROLLED;
        do g.control = (int32_t)q(rng);
        while ((uint32_t)g.control == g.target);
    }
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    // dense, diag(1,d), diag(d0,d1), identity, then the structured classes:
    // real, X, entries +-1/2, Z, sqrt(W)-like, real u00 (U3)
    const int kind = (int)(rng() % 10);
    for (double &x : g.u) x = u(rng);
    if (kind >= 1 && kind <= 3) g.u[2] = g.u[3] = g.u[4] = g.u[5] = 0.0;
    if (kind == 1 || kind == 3) { g.u[0] = 1.0; g.u[1] = 0.0; }
    if (kind == 3) { g.u[6] = 1.0; g.u[7] = 0.0; }
    if (kind == 4) g.u[1] = g.u[3] = g.u[5] = g.u[7] = 0.0;
    if (kind == 5) for (int i = 0; i < 8; ++i) g.u[i] = (i == 2 || i == 4) ? 1.0 : 0.0;
    if (kind == 6) for (double &x : g.u) x = (rng() & 1) ? 0.5 : -0.5;
    if (kind == 7) for (int i = 0; i < 8; ++i) g.u[i] = i == 0 ? 1.0 : i == 6 ? -1.0 : 0.0;
    if (kind == 9) g.u[1] = 0.0;
    if (kind == 8) {
        for (double &x : g.u) x = (rng() & 1) ? 0.5 : -0.5;
        g.u[2] = 0.0;
        g.u[5] = 0.0;
        g.u[3] = u(rng);
        g.u[4] = u(rng);
    }
    return g;
}

static void check_plan(const std::vector<qvg_gate> &ops, const PlanOptions &po) {
    std::vector<qvg_gate> list = ops;
    if (po.reorder) {
        std::vector<uint64_t> order;
        list = reorder_for_tiles(ops.data(), ops.size(), po, &order);
        CHECK(list.size() == ops.size() && order.size() == ops.size());
        // every inverted pair acts on disjoint qubits; in the bit-exact mode
        // one of the two is a permutation or a +-1 phase
        std::vector<uint64_t> pos(ops.size());
        for (uint64_t x = 0; x < order.size(); ++x) pos[order[x]] = x;
        for (uint64_t a = 0; a < ops.size(); ++a)
            for (uint64_t b = a + 1; b < ops.size(); ++b) {
                if (pos[a] < pos[b]) continue;
                const OpInfo oa = classify(ops[a]), ob = classify(ops[b]);
                auto touches = [](const OpInfo &o, int q) { return o.target == q || o.control == q; };
                CHECK(!touches(oa, ob.target) && (ob.control < 0 || !touches(oa, ob.control)));
                if (po.reorder == REORDER_EXACT) CHECK(exact_commuter(oa) || exact_commuter(ob));
            }
    }
    const Plan p = make_plan(list.data(), list.size(), po);
    uint64_t covered = 0, live = 0;
    for (const qvg_gate &g : list) live += classify(g).identity ? 0 : 1;
    for (const Pass &pass : p.passes) {
        if (pass.kind == PASS_PERM) {  // k_tile_perm records: X / sign flips on tile-local bits, op order
            const TileGeom &g = pass.geom;
            CHECK(po.perm && po.classes && g.nrec >= 1 && g.nrec <= kMaxTileRecs && g.ngroups == 0);
            for (int i = 0; i < g.nrec; ++i) {
                const TileOp &t = p.tile_ops[pass.op_begin + i];
                CHECK(t.kind == TILE_PAIR || t.kind == TILE_DIAG);
                CHECK(t.tbit < g.k && t.cbit < g.k && (t.cbit < 0 || t.cbit != t.tbit));
                if (t.kind == TILE_PAIR) CHECK(t.tbit >= 0);
                if (t.tbit < 0) CHECK(t.kind == TILE_DIAG && t.gtgt != 0 && !(t.gtgt & (t.gtgt - 1)));
                if (t.cbit < 0 && t.greq) CHECK(!(t.greq & (t.greq - 1)));
            }
            covered += (uint64_t)g.nrec;
            continue;
        }
        covered += pass.kind == PASS_TILE ? 0 : 1;
        if (pass.kind != PASS_TILE) continue;
        const TileGeom &g = pass.geom;
        CHECK(g.nrec <= kMaxTileRecs && g.nrec >= 2);
        CHECK(g.k <= (int)po.n && g.lowc >= 0 && g.nhi == g.k - g.lowc);
        CHECK(g.sub >= 2 && g.sub <= 5);
        int rec = (int)pass.op_begin, groups = 0;
        const int end = (int)pass.op_begin + g.nrec;
        while (rec < end) {
            const TileOp &h = p.tile_ops[rec];
            CHECK(h.kind == TILE_GROUP);
            for (int s = 0; s < g.sub; ++s) CHECK((int)((h.gtgt >> (8 * s)) & 0xff) < g.k);
            const int nops = h.tbit;
            CHECK(nops >= 1 && rec + 1 + nops <= end);
            for (int i = 0; i < nops; ++i) {
                const TileOp &t = p.tile_ops[rec + 1 + i];
                // record values: 8 doubles, or 8 floats for complex64 passes
                double uv[8];
                for (int e = 0; e < 8; ++e)
                    uv[e] = po.amp_bytes == 8 ? (double)reinterpret_cast<const float *>(t.u)[e] : t.u[e];
                CHECK(t.kind == TILE_PAIR || t.kind == TILE_DIAG);
                if (t.kind == TILE_PAIR) {
                    // 30*class + 6*J + (K+1) with J >= 0 (target in the group); an X-class op may
                    // keep an in-tile control outside the group as a thread-index bit (kSlotCtlTest)
                    CHECK((t.slot & ~(0xff | kSlotCtlTest)) == 0 && (t.slot & 0xff) < kDispDiag);
                    const int pd = t.slot & 0xff;
                    const int cls = pd / 30, js = 8 * ((pd % 30) / 6), pk = (pd % 30) % 6 - 1;
                    if (t.slot & kSlotCtlTest)
                        CHECK(cls == TILE_CLS_SWAP && pk < 0 && t.cbit >= 0 && t.cbit < g.k - g.sub);
                    else
                        CHECK(pk >= 0 || t.cbit < 0);
                    CHECK(cls >= TILE_CLS_GEN && cls <= TILE_CLS_U00R && (po.classes || cls == TILE_CLS_GEN));
                    CHECK((g.cls_set >> cls) & 1);
                    if (cls == TILE_CLS_SQW)  // (s0/2, -s0 s1, q, 0) per row
                        for (int row = 0; row < 2; ++row) {
                            const double *m = uv + 4 * row;
                            CHECK((m[0] == 0.5 || m[0] == -0.5) && (m[1] == 1.0 || m[1] == -1.0) && m[3] == 0.0);
                        }
                    CHECK(js < 8 * g.sub);
                    if (!(js < 8 * g.sub) && failures < 5)
                        std::fprintf(stderr, "  slot %d sub %d k %d tbit %d cbit %d\n", t.slot, g.sub, g.k, t.tbit, t.cbit);
                    if (cls == TILE_CLS_HALF)  // (s0/2, -s0 s1, -s2 s3, s0 s2) per row
                        for (int row = 0; row < 2; ++row) {
                            const double *m = uv + 4 * row;
                            CHECK((m[0] == 0.5 || m[0] == -0.5) && (m[1] == 1.0 || m[1] == -1.0) &&
                                  (m[2] == 1.0 || m[2] == -1.0) && (m[3] == 1.0 || m[3] == -1.0));
                        }
                } else {
                    const int d = t.slot & 0xff;  // 180 + 36*neg + 6*(J+1) + (K+1)
                    CHECK(d >= kDispDiag && d < kDispDiag + 72);
                    const int neg = (d - kDispDiag) / 36, J = ((d - kDispDiag) % 36) / 6 - 1,
                              K = (d - kDispDiag) % 6 - 1;
                    CHECK(J < g.sub && K < g.sub && (J < 0 || J != K));
                    CHECK(po.classes || !neg);
                    if (neg) CHECK(uv[0] == 1.0 && uv[6] == -1.0 && !(t.slot & kSlotD0));
                    CHECK(((t.slot & kSlotT1) != 0) == (J < 0));
                    CHECK(((t.slot & kSlotCtlTest) != 0) == (K < 0 && t.cbit >= 0));
                }
                ++covered;
            }
            rec += 1 + nops;
            ++groups;
        }
        CHECK(groups == g.ngroups);
    }
    CHECK(covered == live);  // every non-identity op exactly once
}

static void check_schedule(const std::vector<qvg_gate> &ops, uint32_t n, uint32_t g, uint32_t kmax) {
    const uint32_t L = n - g;
    QubitMap map;
    map.reset(n);
    std::vector<ShardStep> steps;
    schedule_ops(n, L, ops.data(), ops.size(), map, steps, kmax);
    schedule_canonicalize(n, L, map, steps, kmax);
    CHECK(map.identity());
    for (const ShardStep &st : steps) {
        if (st.type == STEP_LOCAL) {
            CHECK(st.op.target < L);
            if (st.op.kind == QVG_OP_CONTROLLED) CHECK((uint32_t)st.op.control < L && (uint32_t)st.op.control != st.op.target);
            CHECK((st.rank_value & ~st.rank_mask) == 0 && st.rank_mask < (1u << g));
        } else if (st.type == STEP_EXCHANGE) {
            CHECK(st.gpos >= L && st.gpos < n && st.lpos < L);
        } else if (st.type == STEP_MULTI_EXCHANGE) {
            const uint32_t k = st.lpos2;
            CHECK(k >= 2 && k <= 4 && (uint32_t)__builtin_popcount(st.gpos) == k && st.gpos < (1u << g));
            for (uint32_t i = 0; i < k; ++i) {
                CHECK(multi_pos(st, i) >= min_exchange_lpos(L) && multi_pos(st, i) < L);
                for (uint32_t j = 0; j < i; ++j) CHECK(multi_pos(st, i) != multi_pos(st, j));
            }
        } else {
            CHECK(st.type == STEP_LOCAL_SWAP && st.lpos < L && st.lpos2 < L && st.lpos != st.lpos2);
        }
    }
}

int main(int argc, char **argv) {
    const int trials = argc > 1 ? std::atoi(argv[1]) : 300;
    std::mt19937_64 rng(2508);
    for (int t = 0; t < trials; ++t) {
        const uint32_t n = 2 + (uint32_t)(rng() % 29);  // 2..30
        std::vector<qvg_gate> ops(1 + rng() % 400);
        for (auto &g : ops) g = random_gate(rng, n);
        PlanOptions po;
        po.n = n;
        po.amp_bytes = rng() % 2 ? 16 : 8;
        po.fuse = rng() % 8 != 0;
        po.tile_qubits = 5 + (uint32_t)(rng() % 8);
        po.carriers = (uint32_t)(rng() % 5);
        po.sub_bits = 3 + (uint32_t)(rng() % 3);
        po.stage_bits = (uint32_t)(rng() % 4);
        po.reorder = (uint32_t)(rng() % 3);
        po.classes = rng() % 4 != 0;
        po.perm = rng() % 2 == 0;
        check_plan(ops, po);
        const uint32_t g = (uint32_t)(rng() % 4);
        if (n >= g + 2) check_schedule(ops, n, g, 1 + (uint32_t)(rng() % 4));
    }
    std::printf("host_fuzz: %d trials, %d failures\n", trials, failures);
    return failures ? 1 : 0;
}
