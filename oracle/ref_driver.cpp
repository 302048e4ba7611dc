// ref_driver.cpp — TEST INFRASTRUCTURE ONLY. A C-ABI shim over the UNMODIFIED
// reference engine (/root/reference/proj/src, compiled in place by
// oracle/Makefile into oracle/_ref/). Used to (1) generate the golden fixtures
// under tests/golden/ and (2) time the reference's CPU path for bench.py
// (`--impl reference` and the `cpu_baseline` leg). Never on the product path.
//
// Every entry point drives the reference's own public API:
//   random_circuit        reference engine.cpp:177-238
//   simulate_dense        reference dense.cpp:146-163
//   BlockStore::create    reference store.cpp:181-214
//   write_full_state      reference engine.cpp:496-509
//   apply_circuit         reference engine.cpp:86-157
//   read_full_state       reference engine.cpp:483-494
//   BlockStore::norm      reference store.cpp:301-316
//   parse_circuit         reference circuit_io.cpp:68-202 (differential parser tests)
#include <cstdint>
#include <cstring>
#include <exception>
#include <filesystem>
#include <memory>
#include <optional>
#include <string>
#include <algorithm>
#include <unistd.h>

#include "qvsim/circuit_io.hpp"
#include "qvsim/dense.hpp"
#include "qvsim/engine.hpp"
#include "qvsim/error.hpp"
#include "qvsim/store.hpp"

namespace {

struct Gate {  // layout of qvg_gate (include/qvg.h)
    std::uint32_t kind, target;
    std::int32_t control;
    std::uint32_t flags;
    double u[8];
};
static_assert(sizeof(Gate) == 80, "qvg_gate layout");

thread_local std::string g_err;
thread_local std::string g_kind;  // reference error class of the last failure

void note_kind(const std::exception &e) {
    g_kind = dynamic_cast<const qvsim::FormatError *>(&e)       ? "FormatError"
             : dynamic_cast<const qvsim::ValidationError *>(&e) ? "ValidationError"
             : dynamic_cast<const qvsim::ParseError *>(&e)      ? "ParseError"
             : dynamic_cast<const qvsim::CapacityError *>(&e)   ? "CapacityError"
             : dynamic_cast<const qvsim::IoError *>(&e)         ? "IoError"
                                                                 : "Error";
}

qvsim::GateMatrix to_matrix(const double *u) {
    return {qvsim::amp_t{u[0], u[1]}, qvsim::amp_t{u[2], u[3]},
            qvsim::amp_t{u[4], u[5]}, qvsim::amp_t{u[6], u[7]}};
}

// Raw GateOp, as SURVEY §0 notes for ops the parser lacks (CP, U3, Haar):
// the engine only reads kind/matrix/target/control.
qvsim::Circuit to_circuit(std::uint32_t n, const Gate *ops, std::uint64_t count) {
    qvsim::Circuit c;
    c.n_qubits = n;
    c.ops.reserve(count);
    for (std::uint64_t k = 0; k < count; ++k) {
        qvsim::GateOp op;
        op.kind = ops[k].kind ? qvsim::OpKind::controlled : qvsim::OpKind::single;
        op.matrix = to_matrix(ops[k].u);
        op.target = ops[k].target;
        if (ops[k].kind) op.control = static_cast<std::uint32_t>(ops[k].control);
        op.name = ops[k].kind ? "cu" : "u";
        c.ops.push_back(std::move(op));
    }
    return c;
}

void from_op(const qvsim::GateOp &op, Gate &g) {
    std::memset(&g, 0, sizeof(g));
    g.kind = op.kind == qvsim::OpKind::controlled ? 1 : 0;
    g.target = op.target;
    g.control = op.control ? static_cast<std::int32_t>(*op.control) : -1;
    const qvsim::amp_t m[4] = {op.matrix.u00, op.matrix.u01, op.matrix.u10, op.matrix.u11};
    for (int i = 0; i < 4; ++i) {
        g.u[2 * i] = m[i].real();
        g.u[2 * i + 1] = m[i].imag();
    }
}

qvsim::Strategy strategy_of(const char *tag) {
    const auto s = qvsim::parse_strategy(tag ? tag : "paired-cached");
    if (!s) throw qvsim::ValidationError(std::string("unknown strategy ") + tag);
    return *s;
}

template <class F> int guarded(F &&f) {
    try {
        f();
        return 0;
    } catch (const std::exception &e) {
        g_err = e.what();
        note_kind(e);
        return 1;
    }
}

struct Handle {
    qvsim::BlockStore store;
};

}  // namespace

extern "C" {

const char *qvr_last_error() { return g_err.c_str(); }
const char *qvr_last_error_kind() { return g_kind.c_str(); }

// reference random_circuit(n, depth, seed); ops and the serialized text.
int qvr_random_circuit(std::uint32_t n, std::uint32_t depth, std::uint64_t seed,
                       Gate *out, char *text, std::uint64_t text_cap) {
    return guarded([&] {
        const qvsim::Circuit c = qvsim::random_circuit(n, depth, seed);
        for (std::size_t k = 0; k < c.ops.size(); ++k) from_op(c.ops[k], out[k]);
        if (text && text_cap) {
            const std::string s = qvsim::serialize_circuit(c);
            std::strncpy(text, s.c_str(), text_cap - 1);
            text[text_cap - 1] = 0;
        }
    });
}

// reference parse_circuit(text, n_override, strict): on success the ops, the
// qubit count and the reference's own serialization; on ParseError returns 2
// with its line number (reference error.hpp ParseError::line()).
int qvr_parse(const char *text, std::int64_t n_override, int strict, Gate *out, std::uint64_t cap,
              std::uint64_t *count, std::uint32_t *n_out, std::uint64_t *err_line, char *ser,
              std::uint64_t ser_cap) {
    try {
        std::optional<std::uint32_t> ov;
        if (n_override >= 0) ov = static_cast<std::uint32_t>(n_override);
        const qvsim::Circuit c = qvsim::parse_circuit(text, ov, strict != 0);
        *count = c.ops.size();
        *n_out = c.n_qubits;
        for (std::size_t k = 0; k < c.ops.size() && k < cap; ++k) from_op(c.ops[k], out[k]);
        if (ser && ser_cap) {
            const std::string s = qvsim::serialize_circuit(c);
            std::strncpy(ser, s.c_str(), ser_cap - 1);
            ser[ser_cap - 1] = 0;
        }
        return 0;
    } catch (const qvsim::ParseError &e) {
        g_err = e.what();
        *err_line = e.line();
        return 2;
    } catch (const std::exception &e) {
        g_err = e.what();
        return 1;
    }
}

// Dense oracle from |0..0> (n <= 12).
int qvr_simulate_dense(std::uint32_t n, const Gate *ops, std::uint64_t count, double *out) {
    return guarded([&] {
        const qvsim::DenseState s = qvsim::simulate_dense(to_circuit(n, ops, count));
        std::memcpy(out, s.amps.data(), s.amps.size() * sizeof(qvsim::amp_t));
    });
}

// Persistent store for timing: create |init> in `dir`.
void *qvr_store_create(const char *dir, std::uint32_t n, std::uint64_t block_amps,
                       std::uint64_t init_index) {
    void *h = nullptr;
    guarded([&] {
        static std::uint64_t serial = 0;  // distinct files for concurrent stores
        const std::filesystem::path p =
            std::filesystem::path(dir) / ("qvr-" + std::to_string(::getpid()) + "-" +
                                          std::to_string(n) + "-" + std::to_string(serial++) + ".qvs");
        const std::uint64_t ba = std::min<std::uint64_t>(block_amps, std::uint64_t{1} << n);
        auto handle = std::make_unique<Handle>(Handle{qvsim::BlockStore::create(p, n, ba, true)});
        if (init_index != 0) {
            // |b> = X on the set bits; only the two touched blocks change, but
            // use the engine so the store path is the reference's own.
            qvsim::Metrics m;
            qvsim::DenseState zero;
            zero.n_qubits = n;
            zero.amps.assign(std::uint64_t{1} << n, qvsim::amp_t{0.0, 0.0});
            zero.amps[init_index] = qvsim::amp_t{1.0, 0.0};
            qvsim::write_full_state(handle->store, zero, m);
        }
        h = handle.release();
    });
    return h;
}

// An existing QVSV file through the reference's BlockStore::open
// (reference store.cpp:216-245).
void *qvr_store_open(const char *path) {
    void *h = nullptr;
    guarded([&] { h = new Handle{qvsim::BlockStore::open(path)}; });
    return h;
}

// The store's file path (the QVSV file the reference engine streams; read
// back with a memory map for multi-GiB states instead of read_full_state).
int qvr_store_path(void *h, char *out, std::uint64_t cap) {
    return guarded([&] {
        const std::string s = static_cast<Handle *>(h)->store.path().string();
        if (s.size() + 1 > cap) throw qvsim::ValidationError("path buffer too small");
        std::memcpy(out, s.c_str(), s.size() + 1);
    });
}

// Close without deleting the file.
void qvr_store_close(void *h) { delete static_cast<Handle *>(h); }

int qvr_store_load(void *h, const double *amps) {
    return guarded([&] {
        auto *hd = static_cast<Handle *>(h);
        qvsim::DenseState s;
        s.n_qubits = hd->store.n_qubits();
        s.amps.resize(hd->store.n_amps());
        std::memcpy(s.amps.data(), amps, s.amps.size() * sizeof(qvsim::amp_t));
        qvsim::Metrics m;
        qvsim::write_full_state(hd->store, s, m);
    });
}

// apply_circuit with the given engine; wall_ms = Metrics::wall_ms
// (steady clock around apply_circuit, engine.cpp:96-105).
int qvr_store_apply(void *h, const Gate *ops, std::uint64_t count, const char *strategy,
                    std::uint32_t workers, std::uint64_t cache_bytes, double *wall_ms) {
    return guarded([&] {
        auto *hd = static_cast<Handle *>(h);
        qvsim::RunConfig cfg;
        cfg.strategy = strategy_of(strategy);
        cfg.workers = workers;
        cfg.cache_bytes = cache_bytes;
        qvsim::Metrics m;
        qvsim::apply_circuit(hd->store, to_circuit(hd->store.n_qubits(), ops, count), cfg, m);
        if (wall_ms) *wall_ms = m.wall_ms;
    });
}

int qvr_store_read(void *h, double *out) {
    return guarded([&] {
        auto *hd = static_cast<Handle *>(h);
        qvsim::Metrics m;
        const qvsim::DenseState s = qvsim::read_full_state(hd->store, m);
        std::memcpy(out, s.amps.data(), s.amps.size() * sizeof(qvsim::amp_t));
    });
}

int qvr_store_norm(void *h, double *out) {
    return guarded([&] {
        qvsim::Metrics m;
        *out = static_cast<Handle *>(h)->store.norm(m);
    });
}

int qvr_store_sync(void *h) {
    return guarded([&] { static_cast<Handle *>(h)->store.sync(); });
}

void qvr_store_destroy(void *h) {
    auto *hd = static_cast<Handle *>(h);
    if (!hd) return;
    const std::filesystem::path p = hd->store.path();
    delete hd;
    std::error_code ec;
    std::filesystem::remove(p, ec);
}

}  // extern "C"
