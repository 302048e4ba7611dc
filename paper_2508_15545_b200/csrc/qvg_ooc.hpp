// qvg_ooc.hpp — out-of-core segment planner: the paper's
// sliding window over a block store, lifted one level up the hierarchy. The
// state lives in host memory; the device holds a window of 2^w amplitudes.
//
// A segment is a maximal run of consecutive ops whose non-diagonal targets fit
// one window qubit set C (|C| = w): the low `base` qubits (contiguous pieces
// of >= 2^base amplitudes in host memory) plus up to `hmax` high qubits.
// Controls outside C and diagonal targets outside C are constant per chunk
// (the chunk fixes every qubit outside C), exactly like a rank predicate or
// rank phase in the sharded schedule (qvg_schedule.hpp). Each segment streams
// the whole state host -> HBM -> host once, chunk by chunk; choosing C anew
// per segment is free because every segment streams everything anyway.
#pragma once

#include <algorithm>
#include <cstdint>
#include <vector>

#include "qvg.h"
#include "qvg_schedule.hpp"

namespace qvg {

struct OocSegment {
    uint64_t begin = 0, end = 0;  // ops [begin, end)
    int lowc = 0;                 // window bits 0..lowc-1 = qubits 0..lowc-1 (contiguous pieces)
    std::vector<int> hiq;         // window bits lowc.. = these qubits, ascending
    uint64_t outmask = 0;         // qubits outside the window (chunk index bits)
};

// High window qubits per segment: pieces of 2^(w-hmax) amplitudes. Windows of
// >= 2^26 amplitudes keep pieces >= 2^16 (1 MiB c128) and <= 1024 per chunk.
inline uint32_t ooc_hmax(uint32_t w) { return w >= 26 ? std::min<uint32_t>(10, w - 16) : w / 2; }

inline std::vector<OocSegment> plan_ooc(uint32_t n, uint32_t w, const qvg_gate *ops, uint64_t count) {
    std::vector<OocSegment> segs;
    const uint32_t hmax = ooc_hmax(w);
    const uint32_t base = w - hmax;
    uint64_t i = 0;
    while (i < count) {
        std::vector<int> high;
        uint64_t j = i;
        for (; j < count; ++j) {
            const qvg_gate &g = ops[j];
            if (op_is_diag(g) || g.target < base) continue;
            if (std::find(high.begin(), high.end(), (int)g.target) != high.end()) continue;
            if (high.size() == hmax) break;
            high.push_back((int)g.target);
        }
        std::vector<char> inq(n, 0);
        for (uint32_t q = 0; q < base; ++q) inq[q] = 1;
        for (int q : high) inq[q] = 1;
        uint32_t size = base + (uint32_t)high.size();
        for (uint32_t q = base; q < n && size < w; ++q)
            if (!inq[q]) {
                inq[q] = 1;
                ++size;
            }
        OocSegment s;
        s.begin = i;
        s.end = j;
        while (s.lowc < (int)n && inq[s.lowc]) ++s.lowc;
        for (uint32_t q = (uint32_t)s.lowc; q < n; ++q) {
            if (inq[q]) s.hiq.push_back((int)q);
            else s.outmask |= 1ull << q;
        }
        segs.push_back(std::move(s));
        i = j;
    }
    return segs;
}

inline uint64_t pdep_host(uint64_t v, uint64_t mask) {
    uint64_t r = 0;
    for (uint64_t m = mask; m; m &= m - 1) {
        if (v & 1) r |= m & (~m + 1);
        v >>= 1;
    }
    return r;
}

inline uint64_t pext_host(uint64_t v, uint64_t mask) {
    uint64_t r = 0, bit = 1;
    for (uint64_t m = mask; m; m &= m - 1, bit <<= 1)
        if (v & m & (~m + 1)) r |= bit;
    return r;
}

// Window bit of global qubit q, -1 when q is outside the window.
inline int window_bit(const OocSegment &s, uint32_t q) {
    if ((int)q < s.lowc) return (int)q;
    for (size_t i = 0; i < s.hiq.size(); ++i)
        if (s.hiq[i] == (int)q) return s.lowc + (int)i;
    return -1;
}

// The segment's ops as seen by the chunk whose outside bits are `base_off`.
inline void chunk_ops(const OocSegment &s, const qvg_gate *ops, uint64_t base_off, std::vector<qvg_gate> &out) {
    out.clear();
    for (uint64_t k = s.begin; k < s.end; ++k) {
        qvg_gate g = ops[k];
        if (g.kind == QVG_OP_CONTROLLED) {
            const int wc = window_bit(s, (uint32_t)g.control);
            if (wc < 0) {
                if (!((base_off >> g.control) & 1ull)) continue;  // control 0 for this whole chunk
                g.kind = QVG_OP_SINGLE;
                g.control = -1;
            } else {
                g.control = wc;
            }
        }
        const int wt = window_bit(s, g.target);
        if (wt >= 0) {
            g.target = (uint32_t)wt;
            out.push_back(g);
            continue;
        }
        // diagonal op on a qubit outside the window: constant phase d_b
        const bool b = (base_off >> g.target) & 1ull;
        const double dr = b ? g.u[6] : g.u[0], di = b ? g.u[7] : g.u[1];
        if (dr == 1.0 && di == 0.0) continue;
        out.push_back(g.kind == QVG_OP_CONTROLLED ? diag_gate((uint32_t)g.control, 1.0, 0.0, dr, di)
                                                  : diag_gate(0, dr, di, dr, di));
    }
}

}  // namespace qvg
