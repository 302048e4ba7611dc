// qvg_schedule.hpp — host-only schedule for a state sharded over G = 2^g
// ranks. No CUDA; exported through qvg_shard_schedule so the
// logic is testable on CPU (tests/test_shard_schedule.py runs it emulated and
// over gloo).
//
// Layout: rank r owns physical indices [r*2^L, (r+1)*2^L), L = n - g — the
// reference's contiguous Eq. 9 partition (reference parallel.cpp:13-37,
// PAPER.md:146). A logical->physical qubit map lets an exchange leave the
// state permuted instead of swapping back.
//
// Per logical op (target t, control c; physical pt, pc):
//   * local target, local/no control       -> local op
//   * local target, global control         -> local op on ranks whose control bit is 1
//   * diagonal op, global target           -> rank-dependent phase, no communication
//   * non-diagonal op, global target       -> pairwise half-shard exchange that
//     swaps physical qubit pt with local qubit L-1 (the paper's cross-node pair,
//     PAPER.md:156-160), then a local op on L-1.
// Exchanges and local ops only move or combine amplitudes with the reference
// pair formula, so the final state is bit-identical for every G.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "qvg.h"

namespace qvg {

enum ShardStepType : uint32_t { STEP_LOCAL = 0, STEP_EXCHANGE = 1, STEP_LOCAL_SWAP = 2, STEP_MULTI_EXCHANGE = 3 };

// One schedule step; the C layout is qvg_shard_step (include/qvg.h).
// STEP_LOCAL runs `op` (physical local qubits) on ranks with
// (rank & rank_mask) == rank_value; STEP_EXCHANGE swaps global physical qubit
// gpos with local qubit lpos (= L-1); STEP_LOCAL_SWAP swaps local lpos, lpos2.
// STEP_MULTI_EXCHANGE swaps k = lpos2 >= 2 global qubits at once: gpos is
// their mask as rank bits (bit j = physical qubit L + j) and lpos packs the
// local positions they trade with, 8 bits each, in the order of gpos's set
// bits. It is an exchange among the 2^k ranks that differ only in those
// bits: (1 - 2^-k) of each shard moves, against k/2 for k pairwise exchanges.
using ShardStep = qvg_shard_step;

// Local positions of a multi-exchange, in the order of the mask's set bits.
inline uint32_t multi_pos(const ShardStep &st, uint32_t i) { return (st.lpos >> (8 * i)) & 0xffu; }

// Bits of r at the set bits of mask, packed (pext) / spread back (pdep).
inline uint32_t bits_pext(uint32_t r, uint32_t mask) {
    uint32_t out = 0, i = 0;
    for (uint32_t b = 0; b < 32; ++b)
        if ((mask >> b) & 1u) out |= ((r >> b) & 1u) << i++;
    return out;
}
inline uint32_t bits_pdep(uint32_t v, uint32_t mask) {
    uint32_t out = 0, i = 0;
    for (uint32_t b = 0; b < 32; ++b)
        if ((mask >> b) & 1u) out |= ((v >> i++) & 1u) << b;
    return out;
}

// The copy transport's chunk plan for one exchange step on one rank, in issue
// order (the layout is qvg_xchunk, include/qvg.h). Each chunk is one grouped
// send/recv with `partner`: this rank sends the `bytes` at `offset` of its
// shard and receives the partner's chunk of the same index into the same
// place. Chunk i of a rank and chunk i of its partner (same round) carry each
// other's data, so the plan needs no coordination beyond the order.
//   STEP_EXCHANGE (gpos, lpos): a rank whose gpos bit is b sends the
//     amplitudes whose local bit lpos is 1 - b: 2^(L-1-lpos) runs of 2^lpos;
//   STEP_MULTI_EXCHANGE (k qubits): round t = 1 .. 2^k - 1 pairs rank r with
//     r ^ pdep(t, mask); r sends (and receives into) the region whose local
//     bits at the k positions read w ^ t, w = pext(r, mask), in runs of
//     2^min(pos) amplitudes.
// Runs longer than chunk_bytes are split. Used by the NCCL copy transport and
// by virtual shards in exchange mode 0 (qvg_shard.hpp), and exported as
// qvg_exchange_plan for the CPU tests (emulated and over gloo).
struct XChunk {
    uint32_t round;    // 1-based exchange round (pairwise: 1)
    uint32_t partner;  // rank this chunk is traded with
    uint64_t offset;   // byte offset into this rank's shard
    uint64_t bytes;
};

inline std::vector<XChunk> exchange_chunks(uint32_t L, uint32_t S, uint64_t chunk_bytes, uint32_t rank,
                                           const ShardStep &st) {
    std::vector<XChunk> out;
    if (chunk_bytes == 0) throw std::invalid_argument("chunk_bytes must be > 0");
    auto emit = [&](uint32_t round, uint32_t partner, uint64_t off, uint64_t len) {
        for (uint64_t o = 0; o < len; o += chunk_bytes)
            out.push_back(XChunk{round, partner, off + o, std::min<uint64_t>(chunk_bytes, len - o)});
    };
    if (st.type == STEP_EXCHANGE) {
        if (st.gpos < L || st.lpos >= L) throw std::invalid_argument("exchange step: gpos must be global, lpos local");
        const uint32_t bit = 1u << (st.gpos - L);
        const uint64_t sendbit = (rank & bit) ? 0 : 1;
        const uint64_t run = (uint64_t)S << st.lpos;
        const uint64_t nruns = 1ull << (L - 1 - st.lpos);
        for (uint64_t k = 0; k < nruns; ++k) emit(1, rank ^ bit, ((k << 1) | sendbit) * run, run);
        return out;
    }
    if (st.type != STEP_MULTI_EXCHANGE) throw std::invalid_argument("not an exchange step");
    const uint32_t k = st.lpos2, mask = st.gpos;
    if (k < 2 || k > 4 || (uint32_t)__builtin_popcount(mask) != k) throw std::invalid_argument("bad multi-exchange step");
    int pos[4], idx[4] = {0, 1, 2, 3};
    for (uint32_t i = 0; i < k; ++i) {
        pos[i] = (int)multi_pos(st, i);
        if ((uint32_t)pos[i] >= L) throw std::invalid_argument("multi-exchange local position out of range");
    }
    std::sort(idx, idx + k, [&](int a, int b) { return pos[a] < pos[b]; });
    const uint32_t w = bits_pext(rank, mask);
    const int pmin = pos[idx[0]];
    const uint64_t run = (uint64_t)S << pmin;
    const uint64_t nruns = 1ull << (L - k - pmin);
    for (uint32_t t = 1; t < (1u << k); ++t) {
        const uint32_t partner = rank ^ bits_pdep(t, mask);
        const uint32_t v = w ^ t;  // the region this rank sends and receives into
        for (uint64_t r = 0; r < nruns; ++r) {
            uint64_t x = r << pmin;
            for (uint32_t j = 0; j < k; ++j) {
                const uint64_t low = (1ull << pos[idx[j]]) - 1;
                x = ((x & ~low) << 1) | (x & low) | ((uint64_t)((v >> idx[j]) & 1u) << pos[idx[j]]);
            }
            emit(t, partner, x * S, run);
        }
    }
    return out;
}

struct QubitMap {
    std::vector<uint32_t> perm;  // logical -> physical
    std::vector<uint32_t> inv;   // physical -> logical
    void reset(uint32_t n) {
        perm.resize(n);
        inv.resize(n);
        for (uint32_t q = 0; q < n; ++q) perm[q] = inv[q] = q;
    }
    void swap_phys(uint32_t a, uint32_t b) {
        const uint32_t la = inv[a], lb = inv[b];
        inv[a] = lb;
        inv[b] = la;
        perm[la] = b;
        perm[lb] = a;
    }
    bool identity() const {
        for (uint32_t q = 0; q < perm.size(); ++q)
            if (perm[q] != q) return false;
        return true;
    }
};

inline bool op_is_diag(const qvg_gate &g) {
    return g.u[2] == 0.0 && g.u[3] == 0.0 && g.u[4] == 0.0 && g.u[5] == 0.0;
}

inline qvg_gate diag_gate(uint32_t target, double d0r, double d0i, double d1r, double d1i) {
    qvg_gate g{};
    g.kind = QVG_OP_SINGLE;
    g.target = target;
    g.control = -1;
    g.u[0] = d0r; g.u[1] = d0i;
    g.u[6] = d1r; g.u[7] = d1i;
    return g;
}

// Append the steps for logical ops[0..count) to `out`, updating `map`.
// Lowest local qubit an exchange may swap with a global one: the exchanged
// half-shard is 2^(L-1-lpos) blocks of 2^lpos contiguous amplitudes, so this
// keeps blocks large (>= 2^(L/2) amplitudes; >= 2^20 = 16 MiB at L >= 32).
inline uint32_t min_exchange_lpos(uint32_t L) { return std::max<uint32_t>(L > 12 ? L - 12 : 0, L / 2); }

// Local qubit to send global for an exchange: the one among the allowed high
// local positions whose logical qubit is used furthest ahead in the remaining
// ops (Belady). For config 4's layer circuit this cuts exchanges per layer by
// 40% / 23% / 13% at 2 / 4 / 8 shards versus always using L-1.
inline uint32_t pick_victim(uint32_t L, const qvg_gate *ops, uint64_t k, uint64_t count, const QubitMap &map) {
    constexpr uint64_t kLookahead = 1024;
    uint32_t best = L - 1;
    uint64_t best_dist = 0;
    for (uint32_t p = L; p-- > min_exchange_lpos(L);) {
        const uint32_t lq = map.inv[p];
        uint64_t dist = ~0ull;  // unused in the window: furthest
        for (uint64_t j = k; j < count && j < k + kLookahead; ++j) {
            const qvg_gate &o = ops[j];
            if (o.target == lq || (o.kind == QVG_OP_CONTROLLED && (uint32_t)o.control == lq)) {
                dist = j - k;
                break;
            }
        }
        if (dist > best_dist) {
            best = p;
            best_dist = dist;
        }
    }
    return best;
}

// Distance to the next op using logical qubit lq (as target, or as control
// too when any_use), within the lookahead window; ~0 when unused there.
inline uint64_t next_use(uint32_t lq, const qvg_gate *ops, uint64_t k, uint64_t count, bool any_use) {
    constexpr uint64_t kLookahead = 1024;
    for (uint64_t j = k; j < count && j < k + kLookahead; ++j) {
        const qvg_gate &o = ops[j];
        if (o.target == lq && (any_use || !op_is_diag(o))) return j - k;
        if (any_use && o.kind == QVG_OP_CONTROLLED && (uint32_t)o.control == lq) return j - k;
    }
    return ~0ull;
}

// Batched exchange choice at op k (whose target is global): the global qubits
// needed as non-diagonal targets soonest, paired with the local qubits (top
// positions only) used furthest ahead, while each brought-in qubit is needed
// before the qubit it displaces. Returns the (global, local) physical pairs;
// one pair means a plain pairwise exchange is as good.
inline std::vector<std::pair<uint32_t, uint32_t>> pick_batch(uint32_t n, uint32_t L, const qvg_gate *ops, uint64_t k,
                                                             uint64_t count, const QubitMap &map, uint32_t kmax) {
    std::vector<std::pair<uint64_t, uint32_t>> need, vic;
    for (uint32_t p = L; p < n; ++p) {
        const uint64_t d = next_use(map.inv[p], ops, k, count, false);
        if (d != ~0ull) need.push_back({d, p});
    }
    for (uint32_t p = L; p-- > min_exchange_lpos(L);) vic.push_back({next_use(map.inv[p], ops, k, count, true), p});
    std::stable_sort(need.begin(), need.end());
    std::stable_sort(vic.begin(), vic.end(), [](const auto &a, const auto &b) { return a.first > b.first; });
    std::vector<std::pair<uint32_t, uint32_t>> out;
    for (size_t i = 0; i < need.size() && i < vic.size() && out.size() < kmax; ++i) {
        if (i > 0 && !(need[i].first < vic[i].first)) break;
        out.push_back({need[i].second, vic[i].second});
    }
    return out;
}

// kmax: most global qubits one exchange may swap (1 = pairwise exchanges only).
inline void schedule_ops(uint32_t n, uint32_t L, const qvg_gate *ops, uint64_t count, QubitMap &map,
                         std::vector<ShardStep> &out, uint32_t kmax = 1) {
    for (uint64_t k = 0; k < count; ++k) {
        const qvg_gate &g = ops[k];
        const bool ctl = g.kind == QVG_OP_CONTROLLED;
        uint32_t pt = map.perm[g.target];
        const bool diag = op_is_diag(g);
        if (pt >= L && !diag) {
            auto batch = kmax >= 2 ? pick_batch(n, L, ops, k, count, map, std::min<uint32_t>(kmax, 4))
                                   : std::vector<std::pair<uint32_t, uint32_t>>{};
            if (batch.size() >= 2) {
                std::sort(batch.begin(), batch.end());  // mask bit order
                ShardStep ex{};
                ex.type = STEP_MULTI_EXCHANGE;
                for (size_t i = 0; i < batch.size(); ++i) {
                    ex.gpos |= 1u << (batch[i].first - L);
                    ex.lpos |= batch[i].second << (8 * i);
                }
                ex.lpos2 = (uint32_t)batch.size();
                out.push_back(ex);
                for (const auto &pr : batch) map.swap_phys(pr.first, pr.second);
                pt = map.perm[g.target];
            } else {
                const uint32_t lpos = pick_victim(L, ops, k, count, map);
                ShardStep ex{};
                ex.type = STEP_EXCHANGE;
                ex.gpos = pt;
                ex.lpos = lpos;
                out.push_back(ex);
                map.swap_phys(pt, lpos);
                pt = lpos;
            }
        }
        const int32_t pc = ctl ? (int32_t)map.perm[(uint32_t)g.control] : -1;
        ShardStep st{};
        st.type = STEP_LOCAL;
        st.op = g;
        if (pc >= (int32_t)L) {  // control on a global qubit: rank predicate
            st.rank_mask |= 1u << (pc - L);
            st.rank_value |= 1u << (pc - L);
            st.op.kind = QVG_OP_SINGLE;
            st.op.control = -1;
        } else if (ctl) {
            st.op.control = pc;
        }
        if (pt < L) {
            st.op.target = pt;
            out.push_back(st);
            continue;
        }
        // Diagonal op on a global target: amplitude x gets d_b, b = its
        // global target bit (constant per rank). Reference pair formula with
        // u01 = u10 = 0 reduces to d_b * x (plus an exact zero).
        const uint32_t bit = 1u << (pt - L);
        for (uint32_t b = 0; b < 2; ++b) {
            const double dr = b ? g.u[6] : g.u[0], di = b ? g.u[7] : g.u[1];
            if (dr == 1.0 && di == 0.0) continue;
            ShardStep s2 = st;
            s2.rank_mask |= bit;
            s2.rank_value |= b ? bit : 0u;
            if (s2.op.kind == QVG_OP_CONTROLLED) {
                // phase d_b on the amplitudes whose (local) control bit is 1
                s2.op = diag_gate((uint32_t)s2.op.control, 1.0, 0.0, dr, di);
            } else {
                s2.op = diag_gate(0, dr, di, dr, di);  // every local amplitude
            }
            out.push_back(s2);
        }
    }
}

// Steps that bring the map back to the identity (canonical index order).
inline void schedule_canonicalize(uint32_t n, uint32_t L, QubitMap &map, std::vector<ShardStep> &out,
                                  uint32_t kmax = 1) {
    // Batched first: every global position whose logical qubit sits on a
    // high local position trades with it in one multi-exchange (k <= 4).
    if (kmax >= 2) {
        std::vector<std::pair<uint32_t, uint32_t>> batch;
        for (uint32_t p = L; p < n && batch.size() < std::min<uint32_t>(kmax, 4); ++p) {
            if (map.inv[p] == p) continue;
            const uint32_t cur = map.perm[p];
            if (cur < L && cur >= min_exchange_lpos(L)) batch.push_back({p, cur});
        }
        if (batch.size() >= 2) {
            ShardStep ex{};
            ex.type = STEP_MULTI_EXCHANGE;
            for (size_t i = 0; i < batch.size(); ++i) {
                ex.gpos |= 1u << (batch[i].first - L);
                ex.lpos |= batch[i].second << (8 * i);
            }
            ex.lpos2 = (uint32_t)batch.size();
            out.push_back(ex);
            for (const auto &pr : batch) map.swap_phys(pr.first, pr.second);
        }
    }
    auto exchange = [&](uint32_t gpos, uint32_t lpos) {
        if (lpos < min_exchange_lpos(L)) {  // small blocks: move the qubit up first
            ShardStep sw{};
            sw.type = STEP_LOCAL_SWAP;
            sw.lpos = lpos;
            sw.lpos2 = L - 1;
            out.push_back(sw);
            map.swap_phys(lpos, L - 1);
            lpos = L - 1;
        }
        ShardStep ex{};
        ex.type = STEP_EXCHANGE;
        ex.gpos = gpos;
        ex.lpos = lpos;
        out.push_back(ex);
        map.swap_phys(gpos, lpos);
    };
    for (uint32_t p = L; p < n; ++p) {
        if (map.inv[p] == p) continue;
        uint32_t cur = map.perm[p];
        if (cur >= L) {  // logical p sits on another global qubit: route via L-1
            exchange(cur, L - 1);
            cur = L - 1;
        }
        exchange(p, cur);
    }
    for (uint32_t l = 0; l < L; ++l) {
        if (map.inv[l] == l) continue;
        const uint32_t cur = map.perm[l];
        ShardStep sw{};
        sw.type = STEP_LOCAL_SWAP;
        sw.lpos = l;
        sw.lpos2 = cur;
        out.push_back(sw);
        map.swap_phys(l, cur);
    }
}

}  // namespace qvg
