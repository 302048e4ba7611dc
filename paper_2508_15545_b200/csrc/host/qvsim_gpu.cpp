// qvsim_gpu.cpp — host layer: gate library, circuit text, seeded generators,
// BASELINE config circuits, and the GPU engine entry over libqvg's C-ABI.
// Behaviour follows the reference files cited per function.
#include "qvsim_gpu.hpp"

#include <algorithm>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numbers>
#include <sstream>
#include <unordered_map>

namespace qvsim {

namespace {

const amp_t kI{0.0, 1.0};

// e^{i x} evaluated as the reference does: std::exp(i1 * x)
// (reference gates.cpp:57-71, engine.cpp:221-224).
amp_t expi(double x) { return std::exp(kI * x); }

bool finite(const amp_t &a) { return std::isfinite(a.real()) && std::isfinite(a.imag()); }

GateMatrix from_reals(const std::vector<double> &p, std::size_t at = 0) {
    return {amp_t{p[at + 0], p[at + 1]}, amp_t{p[at + 2], p[at + 3]}, amp_t{p[at + 4], p[at + 5]},
            amp_t{p[at + 6], p[at + 7]}};
}

// sqrt of a Hermitian unitary G: (1+i)/2 I + (1-i)/2 G (eigenvalues +-1 -> 1, i).
GateMatrix sqrt_hermitian_unitary(const GateMatrix &g) {
    const amp_t a{0.5, 0.5}, b{0.5, -0.5};
    return {a + b * g.u00, b * g.u01, b * g.u10, a + b * g.u11};
}

void check_unitary(const GateMatrix &g, bool strict, const std::string &what) {
    const double tol = strict ? kBuiltinUnitaryTol : kCustomUnitaryTol;
    const double dev = unitarity_deviation(g);
    if (!(dev <= tol))
        throw ValidationError(what + " is not unitary (deviation " + std::to_string(dev) + " > tolerance " +
                              std::to_string(tol) + ")");
}

}  // namespace

// reference circuit.cpp:15-29
double unitarity_deviation(const GateMatrix &u) {
    if (!finite(u.u00) || !finite(u.u01) || !finite(u.u10) || !finite(u.u11))
        return std::numeric_limits<double>::infinity();
    const amp_t c00 = std::conj(u.u00) * u.u00 + std::conj(u.u10) * u.u10;
    const amp_t c01 = std::conj(u.u00) * u.u01 + std::conj(u.u10) * u.u11;
    const amp_t c10 = std::conj(u.u01) * u.u00 + std::conj(u.u11) * u.u10;
    const amp_t c11 = std::conj(u.u01) * u.u01 + std::conj(u.u11) * u.u11;
    return std::max({std::abs(c00 - 1.0), std::abs(c01), std::abs(c10), std::abs(c11 - 1.0)});
}

// reference circuit.cpp:31-52
std::vector<Violation> validate_circuit(const Circuit &c) {
    std::vector<Violation> out;
    for (std::size_t i = 0; i < c.ops.size(); ++i) {
        const GateOp &op = c.ops[i];
        if (op.target >= c.n_qubits)
            out.push_back({i, "target " + std::to_string(op.target) + " >= n_qubits " + std::to_string(c.n_qubits)});
        if (op.control) {
            if (*op.control >= c.n_qubits)
                out.push_back(
                    {i, "control " + std::to_string(*op.control) + " >= n_qubits " + std::to_string(c.n_qubits)});
            if (*op.control == op.target)
                out.push_back({i, "control equals target (" + std::to_string(op.target) + ")"});
        }
    }
    return out;
}

void check_status(int status) {
    if (status == QVG_OK) return;
    const std::string msg = qvg_last_error();
    switch (status) {
    case QVG_ERR_VALIDATION: throw ValidationError(msg);
    case QVG_ERR_CAPACITY: throw CapacityError(msg);
    case QVG_ERR_FORMAT: throw FormatError(msg);
    default: throw IoError(msg);
    }
}

// ---- gate library -------------------------------------------------------------

std::optional<std::size_t> gate_arity(const std::string &name) {
    static const std::unordered_map<std::string, std::size_t> arity = {
        {"h", 0},  {"x", 0},  {"y", 0},  {"z", 0},  {"s", 0},  {"sdg", 0}, {"t", 0},
        {"tdg", 0}, {"rx", 1}, {"ry", 1}, {"rz", 1}, {"u", 8},  {"p", 1},   {"u3", 3},
        {"sx", 0}, {"sy", 0}, {"sw", 0}};
    const auto it = arity.find(name);
    if (it == arity.end()) return std::nullopt;
    return it->second;
}

const std::vector<std::string> &builtin_gate_names() {
    // The reference's pool, in its order (reference gates.cpp:23-27):
    // random_circuit draws from it, so the order is part of the seed contract.
    static const std::vector<std::string> names = {"h", "x", "y", "z", "s", "sdg", "t", "tdg", "rx", "ry", "rz", "u"};
    return names;
}

// reference gates.cpp:29-93 (+ p, u3, sx, sy, sw)
GateMatrix make_gate(const std::string &name, const std::vector<double> &params, bool strict) {
    const auto arity = gate_arity(name);
    if (!arity) throw ValidationError("unknown gate '" + name + "'");
    if (params.size() != *arity)
        throw ValidationError("gate '" + name + "' expects " + std::to_string(*arity) + " parameter(s), got " +
                              std::to_string(params.size()));
    const double r = 1.0 / std::sqrt(2.0);
    const double pi = std::numbers::pi;
    const amp_t one{1, 0}, zero{0, 0};
    if (name == "h") return {amp_t{r, 0}, amp_t{r, 0}, amp_t{r, 0}, amp_t{-r, 0}};
    if (name == "x") return {zero, one, one, zero};
    if (name == "y") return {zero, amp_t{0, -1}, amp_t{0, 1}, zero};
    if (name == "z") return {one, zero, zero, amp_t{-1, 0}};
    if (name == "s") return {one, zero, zero, amp_t{0, 1}};
    if (name == "sdg") return {one, zero, zero, amp_t{0, -1}};
    if (name == "t") return {one, zero, zero, expi(pi / 4)};
    if (name == "tdg") return {one, zero, zero, expi(-pi / 4)};
    if (name == "rx" || name == "ry") {
        const double c = std::cos(params[0] / 2), s = std::sin(params[0] / 2);
        if (name == "rx") return {amp_t{c, 0}, amp_t{0, -s}, amp_t{0, -s}, amp_t{c, 0}};
        return {amp_t{c, 0}, amp_t{-s, 0}, amp_t{s, 0}, amp_t{c, 0}};
    }
    if (name == "rz") return {expi(-(params[0] / 2)), zero, zero, expi(params[0] / 2)};
    if (name == "p") return {one, zero, zero, expi(params[0])};
    if (name == "u3") {
        const double th = params[0], ph = params[1], la = params[2];
        const double c = std::cos(th / 2), s = std::sin(th / 2);
        return {amp_t{c, 0}, -expi(la) * s, expi(ph) * s, expi(ph + la) * c};
    }
    if (name == "sx") return sqrt_hermitian_unitary(make_gate("x", {}));
    if (name == "sy") return sqrt_hermitian_unitary(make_gate("y", {}));
    if (name == "sw") {
        const GateMatrix w{zero, amp_t{r, -r}, amp_t{r, r}, zero};  // (X + Y)/sqrt 2
        return sqrt_hermitian_unitary(w);
    }
    // "u": 8 reals row-major, checked for unitarity (reference gates.cpp:70-80)
    const GateMatrix g = from_reals(params);
    check_unitary(g, strict, "custom gate");
    return g;
}

GateOp single_op(const std::string &name, std::uint32_t target, std::vector<double> params) {
    GateOp op;
    op.kind = OpKind::single;
    op.matrix = make_gate(name, params);
    op.target = target;
    op.name = name;
    op.params = std::move(params);
    return op;
}

GateOp controlled_op(const std::string &name, std::uint32_t control, std::uint32_t target,
                     std::vector<double> params) {
    GateOp op;
    op.kind = OpKind::controlled;
    op.target = target;
    op.control = control;
    op.name = name;
    if (name == "cx" || name == "cz") {
        if (!params.empty()) throw ValidationError("'" + name + "' takes no parameters");
        op.matrix = make_gate(name == "cx" ? "x" : "z", {});
    } else if (name == "cp") {
        if (params.size() != 1) throw ValidationError("'cp' expects 1 parameter");
        op.matrix = make_gate("p", params);
    } else if (name == "cu") {
        if (params.size() != 8) throw ValidationError("'cu' expects 8 parameters");
        op.matrix = make_gate("u", params);
    } else {
        throw ValidationError("unknown controlled gate '" + name + "'");
    }
    op.params = std::move(params);
    return op;
}

// ---- circuit text (reference circuit_io.cpp:15-202) ---------------------------

namespace {

std::vector<std::string> tokens_of(std::string_view line) {
    if (const auto hash = line.find('#'); hash != std::string_view::npos) line = line.substr(0, hash);
    std::vector<std::string> out;
    std::istringstream in{std::string(line)};
    for (std::string t; in >> t;) out.push_back(t);
    return out;
}

std::uint32_t qubit_of(const std::string &tok, std::size_t line) {
    std::size_t used = 0;
    unsigned long v = 0;
    bool ok = !tok.empty() && tok[0] != '-';
    if (ok) {
        try {
            v = std::stoul(tok, &used);
        } catch (const std::exception &) {
            ok = false;
        }
    }
    if (!ok || used != tok.size()) throw ParseError(line, "expected a qubit index, got '" + tok + "'");
    return static_cast<std::uint32_t>(v);
}

double real_of(const std::string &tok, std::size_t line) {
    std::size_t used = 0;
    double v = 0;
    try {
        v = std::stod(tok, &used);
    } catch (const std::exception &) {
        throw ParseError(line, "expected a number, got '" + tok + "'");
    }
    if (used != tok.size()) throw ParseError(line, "expected a number, got '" + tok + "'");
    if (!std::isfinite(v)) throw ParseError(line, "number must be finite, got '" + tok + "'");
    return v;
}

std::string real17(double v) {
    char buf[32];
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return buf;
}

std::size_t controlled_arity(const std::string &m) {
    if (m == "cx" || m == "cz") return 0;
    if (m == "cp") return 1;
    if (m == "cu") return 8;
    return ~std::size_t{0};
}

}  // namespace

Circuit parse_circuit(std::string_view text, std::optional<std::uint32_t> n_override, bool strict) {
    std::optional<std::uint32_t> declared;
    std::vector<std::pair<GateOp, std::size_t>> ops;
    std::size_t line_no = 0, pos = 0;
    while (pos <= text.size()) {
        const std::size_t nl = text.find('\n', pos);
        const std::string_view line = text.substr(pos, nl == std::string_view::npos ? std::string_view::npos : nl - pos);
        pos = nl == std::string_view::npos ? text.size() + 1 : nl + 1;
        ++line_no;
        const auto tok = tokens_of(line);
        if (tok.empty()) continue;
        const std::string &m = tok[0];
        if (m == "qubits") {
            if (declared || !ops.empty())
                throw ParseError(line_no, "'qubits' directive must appear once, before any instruction");
            if (tok.size() != 2) throw ParseError(line_no, "'qubits' takes one argument");
            const std::uint32_t n = qubit_of(tok[1], line_no);
            if (n == 0) throw ParseError(line_no, "qubit count must be positive");
            declared = n;
            continue;
        }
        if (m == "swap") {
            // SWAP(a, b) = CX(a,b) CX(b,a) CX(a,b), the decomposition config 1's
            // bit reversal uses; it serializes as those three cx lines
            // (SURVEY §8f row 4).
            if (tok.size() != 3) throw ParseError(line_no, "'swap' takes <qubit> <qubit>");
            const std::uint32_t a = qubit_of(tok[1], line_no), b = qubit_of(tok[2], line_no);
            if (a == b) throw ParseError(line_no, "swap of a qubit with itself (" + std::to_string(a) + ")");
            ops.emplace_back(controlled_op("cx", a, b), line_no);
            ops.emplace_back(controlled_op("cx", b, a), line_no);
            ops.emplace_back(controlled_op("cx", a, b), line_no);
            continue;
        }
        if (const std::size_t ca = controlled_arity(m); ca != ~std::size_t{0}) {
            if (tok.size() != 3 + ca)
                throw ParseError(line_no, "'" + m + "' takes <control> <target>" +
                                              (ca ? " and " + std::to_string(ca) + " number(s)" : std::string()));
            const std::uint32_t c = qubit_of(tok[1], line_no), t = qubit_of(tok[2], line_no);
            if (c == t) throw ParseError(line_no, "control equals target (" + std::to_string(t) + ")");
            std::vector<double> params;
            for (std::size_t i = 0; i < ca; ++i) params.push_back(real_of(tok[3 + i], line_no));
            try {
                ops.emplace_back(controlled_op(m, c, t, std::move(params)), line_no);
            } catch (const ValidationError &e) {
                throw ParseError(line_no, e.what());
            }
            continue;
        }
        const auto arity = gate_arity(m);
        if (!arity) throw ParseError(line_no, "unknown instruction '" + m + "'");
        if (tok.size() != 2 + *arity)
            throw ParseError(line_no, "'" + m + "' takes <qubit> and " + std::to_string(*arity) +
                                          " number(s), got " + std::to_string(tok.size() - 1) + " argument(s)");
        const std::uint32_t t = qubit_of(tok[1], line_no);
        std::vector<double> params;
        for (std::size_t i = 0; i < *arity; ++i) params.push_back(real_of(tok[2 + i], line_no));
        GateOp op;
        try {
            op = single_op(m, t, params);
            if (m == "u" && strict) make_gate("u", params, true);
        } catch (const ValidationError &e) {
            throw ParseError(line_no, e.what());
        }
        ops.emplace_back(std::move(op), line_no);
    }
    if (declared && n_override && *declared != *n_override)
        throw ParseError(1, "declared qubit count " + std::to_string(*declared) + " conflicts with requested " +
                                std::to_string(*n_override));
    const auto n = declared ? declared : n_override;
    if (!n) throw ParseError(1, "qubit count unspecified: add a 'qubits <n>' directive or pass one explicitly");
    Circuit c;
    c.n_qubits = *n;
    for (auto &[op, ln] : ops) c.ops.push_back(std::move(op));
    if (const auto v = validate_circuit(c); !v.empty()) throw ParseError(ops[v.front().op_index].second, v.front().message);
    return c;
}

std::string serialize_circuit(const Circuit &c) {
    std::string out = "qubits " + std::to_string(c.n_qubits) + "\n";
    for (const GateOp &op : c.ops) {
        out += op.name;
        if (op.control) out += " " + std::to_string(*op.control);
        out += " " + std::to_string(op.target);
        for (double p : op.params) out += " " + real17(p);
        out += "\n";
    }
    return out;
}

// ---- generators -----------------------------------------------------------------

// reference engine.cpp:159-171: reject below 2^64 mod bound.
std::uint64_t uniform_below(std::mt19937_64 &rng, std::uint64_t bound) {
    if (bound == 0) throw ValidationError("uniform_below: bound must be positive");
    const std::uint64_t reject = (0 - bound) % bound;
    std::uint64_t r;
    do r = rng();
    while (r < reject);
    return r % bound;
}

// reference engine.cpp:173-175
double uniform_unit(std::mt19937_64 &rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

// reference engine.cpp:177-232 (same draw order, same matrix expressions).
Circuit random_circuit(std::mt19937_64 &rng, std::uint32_t n, std::uint32_t depth) {
    if (n < 1) throw ValidationError("circuit needs at least one qubit");
    std::vector<std::string> pool = builtin_gate_names();
    if (n >= 2) {
        pool.push_back("cx");
        pool.push_back("cz");
    }
    const double tau = 2.0 * std::numbers::pi;
    Circuit c;
    c.n_qubits = n;
    c.ops.reserve(depth);
    for (std::uint32_t k = 0; k < depth; ++k) {
        const std::string &name = pool[uniform_below(rng, pool.size())];
        const auto t = static_cast<std::uint32_t>(uniform_below(rng, n));
        if (name == "cx" || name == "cz") {
            auto ctl = static_cast<std::uint32_t>(uniform_below(rng, n - 1));
            ctl += ctl >= t ? 1 : 0;
            c.ops.push_back(controlled_op(name, ctl, t));
            continue;
        }
        const std::size_t arity = *gate_arity(name);
        if (arity == 0) {
            c.ops.push_back(single_op(name, t));
        } else if (arity == 1) {
            c.ops.push_back(single_op(name, t, {tau * uniform_unit(rng)}));
        } else {
            // global phase x Rz x Ry x Rz, exactly unitary for any angles
            const double phi = tau * uniform_unit(rng);
            const double beta = tau * uniform_unit(rng);
            const double gamma = tau * uniform_unit(rng);
            const double delta = tau * uniform_unit(rng);
            const double cg = std::cos(gamma / 2), sg = std::sin(gamma / 2);
            const amp_t a = std::exp(kI * (phi - beta / 2 - delta / 2)) * cg;
            const amp_t b = -std::exp(kI * (phi - beta / 2 + delta / 2)) * sg;
            const amp_t d = std::exp(kI * (phi + beta / 2 - delta / 2)) * sg;
            const amp_t e = std::exp(kI * (phi + beta / 2 + delta / 2)) * cg;
            c.ops.push_back(single_op(name, t, {a.real(), a.imag(), b.real(), b.imag(), d.real(), d.imag(),
                                                e.real(), e.imag()}));
        }
    }
    return c;
}

Circuit random_circuit(std::uint32_t n, std::uint32_t depth, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    return random_circuit(rng, n, depth);
}

// reference engine.cpp:240-251
Circuit make_benchmark_circuit(std::uint32_t n) {
    if (n < 1) throw ValidationError("circuit needs at least one qubit");
    Circuit c;
    c.n_qubits = n;
    for (std::uint32_t k = 0; k < n; ++k) c.ops.push_back(single_op("h", k));
    return c;
}

// ---- BASELINE configs -------------------------------------------------------------

Circuit u3_ladder_circuit(std::uint32_t n, std::uint32_t layers, std::uint64_t seed) {
    if (n < 2) throw ValidationError("u3 ladder needs at least two qubits");
    std::mt19937_64 rng(seed);
    const double tau = 2.0 * std::numbers::pi;
    Circuit c;
    c.n_qubits = n;
    c.ops.reserve((std::size_t)layers * (2 * n - 1));
    for (std::uint32_t l = 0; l < layers; ++l) {
        for (std::uint32_t q = 0; q < n; ++q) {
            const double th = tau * uniform_unit(rng);
            const double ph = tau * uniform_unit(rng);
            const double la = tau * uniform_unit(rng);
            c.ops.push_back(single_op("u3", q, {th, ph, la}));
        }
        for (std::uint32_t q = 0; q + 1 < n; ++q) c.ops.push_back(controlled_op("cx", q, q + 1));
    }
    return c;
}

Circuit qft_circuit(std::uint32_t n, std::uint64_t seed, std::uint64_t *basis_index, bool h_layer) {
    if (n < 1 || n > 63) throw ValidationError("qft needs 1..63 qubits");
    std::mt19937_64 rng(seed);
    const std::uint64_t b = uniform_below(rng, std::uint64_t{1} << n);
    if (basis_index) *basis_index = b;
    Circuit c;
    c.n_qubits = n;
    for (std::uint32_t q = 0; q < n; ++q)
        if ((b >> q) & 1u) c.ops.push_back(single_op("x", q));
    if (h_layer)
        for (std::uint32_t q = 0; q < n; ++q) c.ops.push_back(single_op("h", q));
    for (std::int64_t t = n - 1; t >= 0; --t) {
        c.ops.push_back(single_op("h", (std::uint32_t)t));
        for (std::int64_t ctl = t - 1; ctl >= 0; --ctl) {
            const double theta = 2.0 * std::numbers::pi / std::ldexp(1.0, (int)(t - ctl + 1));
            c.ops.push_back(controlled_op("cp", (std::uint32_t)ctl, (std::uint32_t)t, {theta}));
        }
    }
    for (std::uint32_t q = 0; q < n / 2; ++q) {  // SWAP(q, n-1-q) = 3 CX
        const std::uint32_t a = q, z = n - 1 - q;
        c.ops.push_back(controlled_op("cx", a, z));
        c.ops.push_back(controlled_op("cx", z, a));
        c.ops.push_back(controlled_op("cx", a, z));
    }
    return c;
}

Circuit haar_sweep_circuit(std::uint32_t n, std::uint64_t seed) {
    if (n < 2) throw ValidationError("haar sweep needs at least two qubits");
    std::mt19937_64 rng(seed);
    auto gaussian = [&]() {  // one complex normal via Box-Muller
        const double u1 = 1.0 - uniform_unit(rng);  // (0, 1]
        const double u2 = uniform_unit(rng);
        const double rad = std::sqrt(-2.0 * std::log(u1));
        return amp_t{rad * std::cos(2.0 * std::numbers::pi * u2), rad * std::sin(2.0 * std::numbers::pi * u2)};
    };
    Circuit c;
    c.n_qubits = n;
    for (std::uint32_t q = 0; q < n; ++q) {
        const amp_t z00 = gaussian(), z01 = gaussian(), z10 = gaussian(), z11 = gaussian();
        // QR by Gram-Schmidt: R's diagonal is real positive, so Q is Haar.
        const double n0 = std::sqrt(std::norm(z00) + std::norm(z10));
        const amp_t q00 = z00 / n0, q10 = z10 / n0;
        const amp_t proj = std::conj(q00) * z01 + std::conj(q10) * z11;
        const amp_t v0 = z01 - proj * q00, v1 = z11 - proj * q10;
        const double n1 = std::sqrt(std::norm(v0) + std::norm(v1));
        const amp_t q01 = v0 / n1, q11 = v1 / n1;
        c.ops.push_back(single_op("u", q, {q00.real(), q00.imag(), q01.real(), q01.imag(), q10.real(), q10.imag(),
                                           q11.real(), q11.imag()}));
    }
    for (std::uint32_t ctl = 0; ctl < n; ++ctl)
        for (std::uint32_t t = 0; t < n; ++t) {
            const std::uint32_t d = ctl > t ? ctl - t : t - ctl;
            if (d == 1 || d == 15 || d == 29) c.ops.push_back(controlled_op("cx", ctl, t));
        }
    return c;
}

Circuit grid_circuit(std::uint32_t rows, std::uint32_t cols, std::uint32_t cycles, std::uint64_t seed) {
    const std::uint32_t n = rows * cols;
    if (rows < 1 || cols < 1 || n < 2) throw ValidationError("grid needs at least two qubits");
    std::mt19937_64 rng(seed);
    static const char *names[3] = {"sx", "sy", "sw"};
    std::vector<int> prev(n, -1);
    Circuit c;
    c.n_qubits = n;
    for (std::uint32_t cy = 0; cy < cycles; ++cy) {
        for (std::uint32_t q = 0; q < n; ++q) {
            int g;
            if (prev[q] < 0) {
                g = (int)uniform_below(rng, 3);
            } else {
                g = (int)uniform_below(rng, 2);
                g += g >= prev[q] ? 1 : 0;  // never repeat the previous draw
            }
            prev[q] = g;
            c.ops.push_back(single_op(names[g], q));
        }
        const std::uint32_t pat = cy % 4;
        for (std::uint32_t r = 0; r < rows; ++r)
            for (std::uint32_t k = 0; k < cols; ++k) {
                const std::uint32_t q = r * cols + k;
                if (pat < 2 && k + 1 < cols && (k % 2) == pat) c.ops.push_back(controlled_op("cz", q, q + 1));
                if (pat >= 2 && r + 1 < rows && (r % 2) == pat - 2) c.ops.push_back(controlled_op("cz", q, q + cols));
            }
    }
    return c;
}

std::vector<qvg_gate> to_gates(const Circuit &c) {
    std::vector<qvg_gate> out(c.ops.size());
    for (std::size_t k = 0; k < c.ops.size(); ++k) {
        const GateOp &op = c.ops[k];
        qvg_gate &g = out[k];
        std::memset(&g, 0, sizeof(g));
        g.kind = op.kind == OpKind::controlled ? QVG_OP_CONTROLLED : QVG_OP_SINGLE;
        g.target = op.target;
        g.control = op.control ? static_cast<std::int32_t>(*op.control) : -1;
        const amp_t m[4] = {op.matrix.u00, op.matrix.u01, op.matrix.u10, op.matrix.u11};
        for (int i = 0; i < 4; ++i) {
            g.u[2 * i] = m[i].real();
            g.u[2 * i + 1] = m[i].imag();
        }
    }
    return out;
}

Circuit from_gates(std::uint32_t n, const qvg_gate *ops, std::size_t count) {
    Circuit c;
    c.n_qubits = n;
    for (std::size_t k = 0; k < count; ++k) {
        const qvg_gate &g = ops[k];
        GateOp op;
        op.kind = g.kind == QVG_OP_CONTROLLED ? OpKind::controlled : OpKind::single;
        op.target = g.target;
        if (g.kind == QVG_OP_CONTROLLED) op.control = static_cast<std::uint32_t>(g.control);
        op.matrix = {amp_t{g.u[0], g.u[1]}, amp_t{g.u[2], g.u[3]}, amp_t{g.u[4], g.u[5]}, amp_t{g.u[6], g.u[7]}};
        op.name = op.control ? "cu" : "u";
        op.params.assign(g.u, g.u + 8);
        c.ops.push_back(std::move(op));
    }
    return c;
}

// ---- engine -----------------------------------------------------------------------

const char *strategy_tag(Strategy s) {
    switch (s) {
    case Strategy::dense: return "dense";
    case Strategy::paired: return "paired";
    case Strategy::paired_cached: return "paired-cached";
    case Strategy::paired_cached_parallel: return "paired-cached-parallel";
    case Strategy::gpu: return "gpu";
    }
    return "unknown";
}

const std::vector<std::string> &strategy_tags() {
    static const std::vector<std::string> tags = {"dense", "paired", "paired-cached", "paired-cached-parallel", "gpu"};
    return tags;
}

std::optional<Strategy> parse_strategy(std::string_view tag) {
    const auto &tags = strategy_tags();
    for (std::size_t i = 0; i < tags.size(); ++i)
        if (tags[i] == tag) return static_cast<Strategy>(i);
    return std::nullopt;
}

StateVector::StateVector(qvg_state *s) : s_(s) {
    check_status(qvg_info(s_, &n_, &precision_, &rank_, &world_));
}

StateVector StateVector::create(std::uint32_t n, std::uint32_t precision, int device) {
    qvg_state *s = nullptr;
    check_status(qvg_create(n, precision, device, &s));
    return StateVector(s);
}

StateVector StateVector::create_sharded(std::uint32_t n, std::uint32_t precision, int device, std::uint32_t rank,
                                        std::uint32_t world, const void *nccl_id) {
    qvg_state *s = nullptr;
    check_status(qvg_create_sharded(n, precision, device, rank, world, nccl_id, &s));
    return StateVector(s);
}

StateVector::StateVector(StateVector &&o) noexcept
    : s_(o.s_), n_(o.n_), precision_(o.precision_), rank_(o.rank_), world_(o.world_) {
    o.s_ = nullptr;
}

StateVector &StateVector::operator=(StateVector &&o) noexcept {
    if (this != &o) {
        if (s_) qvg_destroy(s_);
        s_ = o.s_;
        n_ = o.n_;
        precision_ = o.precision_;
        rank_ = o.rank_;
        world_ = o.world_;
        o.s_ = nullptr;
    }
    return *this;
}

StateVector::~StateVector() {
    if (s_) qvg_destroy(s_);
}

void StateVector::init_basis(std::uint64_t index) { check_status(qvg_init_basis(s_, index)); }

void StateVector::load(const amp_t *amps, std::uint64_t offset, std::uint64_t count) {
    if (precision_ == QVG_C128) {
        check_status(qvg_load(s_, amps, offset, count));
        return;
    }
    std::vector<float> f(2 * count);
    for (std::uint64_t i = 0; i < count; ++i) {
        f[2 * i] = (float)amps[i].real();
        f[2 * i + 1] = (float)amps[i].imag();
    }
    check_status(qvg_load(s_, f.data(), offset, count));
}

void StateVector::read(amp_t *out, std::uint64_t offset, std::uint64_t count) const {
    if (precision_ == QVG_C128) {
        check_status(qvg_read(s_, out, offset, count));
        return;
    }
    std::vector<float> f(2 * count);
    check_status(qvg_read(s_, f.data(), offset, count));
    for (std::uint64_t i = 0; i < count; ++i) out[i] = amp_t{f[2 * i], f[2 * i + 1]};
}

amp_t StateVector::amplitude(std::uint64_t index) const {
    if (index >= n_amps()) throw ValidationError("amplitude index " + std::to_string(index) + " out of range");
    amp_t a;
    read(&a, index, 1);
    return a;
}

double StateVector::norm() const {
    double v = 0.0;
    check_status(qvg_norm(s_, &v));
    return v;
}

void StateVector::probabilities(double *out, std::uint64_t offset, std::uint64_t count) const {
    check_status(qvg_probabilities(s_, out, offset, count));
}

std::vector<std::pair<std::uint64_t, amp_t>> StateVector::top_amplitudes(std::size_t k) const {
    std::vector<std::pair<std::uint64_t, amp_t>> out;
    if (k == 0) return out;
    const std::size_t kk = (std::size_t)std::min<std::uint64_t>(k, n_amps());
    std::vector<std::uint64_t> idx(kk);
    std::vector<double> amps(2 * kk);
    check_status(qvg_top_amplitudes(s_, (std::uint32_t)kk, idx.data(), amps.data()));
    for (std::size_t i = 0; i < kk; ++i) out.emplace_back(idx[i], amp_t{amps[2 * i], amps[2 * i + 1]});
    return out;
}

void StateVector::set_option(int key, std::int64_t value) { check_status(qvg_set_option(s_, key, value)); }

qvg_stats StateVector::stats() const {
    qvg_stats st{};
    check_status(qvg_stats_get(s_, &st));
    return st;
}

void StateVector::sync() const { check_status(qvg_sync(s_)); }

void apply_circuit(StateVector &state, const Circuit &circuit, const RunConfig &config, Metrics &metrics) {
    // reference engine.cpp:58-71 check_match
    if (circuit.n_qubits != state.n_qubits())
        throw ValidationError("circuit is for " + std::to_string(circuit.n_qubits) + " qubits, state holds " +
                              std::to_string(state.n_qubits()));
    if (const auto v = validate_circuit(circuit); !v.empty())
        throw ValidationError("invalid circuit: op " + std::to_string(v.front().op_index) + ": " + v.front().message);
    if (config.strategy != Strategy::gpu)
        throw ValidationError(std::string("strategy '") + strategy_tag(config.strategy) +
                              "' runs on the reference's block-store engine; a device state takes 'gpu'");
    metrics.strategy = strategy_tag(config.strategy);
    metrics.workers = state.world();
    metrics.peak_cache_bytes = std::max<std::uint64_t>(
        metrics.peak_cache_bytes, (std::uint64_t)(state.precision() == 128 ? 16 : 8) << (state.n_qubits() - std::countr_zero(state.world())));
    const double before = metrics.wall_ms;
    const auto t0 = std::chrono::steady_clock::now();
    const qvg_stats s0 = state.stats();
    auto stamp = [&] {
        metrics.wall_ms =
            before + std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        const qvg_stats s1 = state.stats();
        metrics.traversals += s1.passes - s0.passes;
        metrics.fused_passes += s1.fused_passes - s0.fused_passes;
        metrics.bytes_moved += s1.bytes_moved - s0.bytes_moved;
        metrics.exchange_bytes += s1.exchange_bytes - s0.exchange_bytes;
        metrics.exchanges += s1.exchanges - s0.exchanges;
        metrics.gates_applied += s1.gates_applied - s0.gates_applied;
    };
    try {
        state.set_option(QVG_OPT_FUSE, config.fuse ? 1 : 0);
        if (config.tile_qubits) state.set_option(QVG_OPT_TILE_QUBITS, config.tile_qubits);
        const std::vector<qvg_gate> gates = to_gates(circuit);
        check_status(qvg_apply(state.handle(), gates.data(), gates.size()));
        if (config.sync) state.sync();
    } catch (...) {
        stamp();
        throw;
    }
    stamp();
}

// ---- verification (reference engine.cpp:253-340) -----------------------------------

namespace {

// reference engine.cpp:77-82
std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// One device configuration run on ops[0..count) from |0...0>, read back.
std::vector<amp_t> run_config(const std::string &cfg, std::uint32_t n, const std::vector<qvg_gate> &ops,
                              std::size_t count, int device) {
    std::vector<amp_t> out(std::size_t{1} << n);
    if (cfg == "out-of-core") {
        out.assign(out.size(), amp_t{0.0, 0.0});
        out[0] = amp_t{1.0, 0.0};
        qvg_stats st{};
        check_status(qvg_apply_host(out.data(), n, 128, device, std::max<std::uint32_t>(4, n - 2), ops.data(), count,
                                    &st));
        return out;
    }
    std::uint32_t shards = 1;
    if (cfg == "shards-2") shards = 2;
    if (cfg == "shards-4") shards = 4;
    StateVector sv = shards == 1 ? StateVector::create(n, 128, device)
                                 : StateVector::create_sharded(n, 128, device, 0, shards, nullptr);
    sv.set_option(QVG_OPT_FUSE, cfg == "per-gate" ? 0 : 1);
    if (cfg == "fused-k5") sv.set_option(QVG_OPT_TILE_QUBITS, 5);
    check_status(qvg_apply(sv.handle(), ops.data(), count));
    sv.read(out.data(), 0, out.size());
    return out;
}

double max_dev(const std::vector<amp_t> &a, const std::vector<amp_t> &b) {
    double m = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        const double d = std::abs(a[i] - b[i]);
        if (!(d <= m)) m = d;  // NaN propagates
    }
    return m;
}

}  // namespace

VerifyResult verify_equivalence(const VerifyOptions &opts) {
    if (opts.min_qubits < 1 || opts.min_qubits > opts.max_qubits)
        throw ValidationError("verify: qubit range must satisfy 1 <= min <= max");
    if (opts.max_qubits > 24) throw ValidationError("verify: max qubits must be <= 24 (states are read back)");
    if (opts.max_depth < 1) throw ValidationError("verify: depth must be >= 1");
    VerifyResult result;
    result.trials = opts.trials;
    for (std::uint64_t trial = 0; trial < opts.trials; ++trial) {
        std::mt19937_64 rng(splitmix64(opts.seed ^ (0x9e3779b97f4a7c15ull * (trial + 1))));
        const auto n = static_cast<std::uint32_t>(opts.min_qubits +
                                                  uniform_below(rng, opts.max_qubits - opts.min_qubits + 1));
        const auto depth = static_cast<std::uint32_t>(1 + uniform_below(rng, opts.max_depth));
        const Circuit circuit = random_circuit(rng, n, depth);
        const std::vector<qvg_gate> ops = to_gates(circuit);
        const std::vector<amp_t> reference = run_config("per-gate", n, ops, ops.size(), opts.device);
        std::vector<std::string> configs = {"fused"};
        if (n >= 5) configs.push_back("fused-k5");
        if (n >= 3) configs.push_back("shards-2");
        if (n >= 4) configs.push_back("shards-4");
        if (n >= 6) configs.push_back("out-of-core");
        for (const std::string &cfg : configs) {
            const double dev = max_dev(reference, run_config(cfg, n, ops, ops.size(), opts.device));
            result.comparisons += 1;
            if (!(dev <= result.max_deviation)) result.max_deviation = dev;
            if (dev <= opts.tolerance) continue;
            VerifyFailure f;
            f.trial = trial;
            f.n_qubits = n;
            f.depth = depth;
            f.config = cfg;
            f.deviation = dev;
            for (std::size_t k = 1; k <= ops.size(); ++k) {  // first divergent prefix
                if (!(max_dev(run_config("per-gate", n, ops, k, opts.device), run_config(cfg, n, ops, k, opts.device)) <=
                      opts.tolerance)) {
                    f.first_divergent_gate = k - 1;
                    break;
                }
            }
            result.failures.push_back(std::move(f));
        }
    }
    return result;
}

}  // namespace qvsim
