// qvsim_gpu.hpp — C++ host layer above the C-ABI (include/qvg.h).
//
// Mirrors the public API of the QVecOpt reference (namespace qvsim,
// /root/reference/proj/include/qvsim/*.hpp) for the gate-application path, so
// a caller of the reference finds the same names, argument meanings and error
// types, and adds Strategy::gpu (reference engine.hpp:21-33 lists the CPU
// strategies). State lives in HBM (StateVector) instead of a block file.
#pragma once

#include <complex>
#include <cstdint>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "qvg.h"

namespace qvsim {

// ---- core types (reference types.hpp:13-68) --------------------------------
using amp_t = std::complex<double>;
inline constexpr std::uint64_t kAmpBytes = 16;

constexpr std::uint64_t pair_index(std::uint64_t i, std::uint32_t k) noexcept {
    return i ^ (std::uint64_t{1} << k);
}
constexpr bool is_pair_base(std::uint64_t i, std::uint32_t k) noexcept { return ((i >> k) & 1u) == 0; }

struct GateMatrix {
    amp_t u00{}, u01{}, u10{}, u11{};
    bool operator==(const GateMatrix &) const = default;
};

double unitarity_deviation(const GateMatrix &u);

enum class OpKind { single, controlled };

struct GateOp {
    OpKind kind = OpKind::single;
    GateMatrix matrix{};
    std::uint32_t target = 0;
    std::optional<std::uint32_t> control;
    std::string name;
    std::vector<double> params;
    bool operator==(const GateOp &) const = default;
};

struct Circuit {
    std::uint32_t n_qubits = 0;
    std::vector<GateOp> ops;
    bool operator==(const Circuit &) const = default;
};

struct Violation {
    std::size_t op_index = 0;
    std::string message;
};

std::vector<Violation> validate_circuit(const Circuit &c);

// ---- errors (reference error.hpp:10-50) ---------------------------------------
class Error : public std::runtime_error {
  public:
    explicit Error(const std::string &what) : std::runtime_error(what) {}
};
class IoError : public Error { using Error::Error; };
class FormatError : public Error { using Error::Error; };
class ParseError : public Error {
  public:
    ParseError(std::size_t line, const std::string &what)
        : Error("line " + std::to_string(line) + ": " + what), line_(line) {}
    std::size_t line() const noexcept { return line_; }

  private:
    std::size_t line_;
};
class CapacityError : public Error { using Error::Error; };
class OracleLimitError : public Error { using Error::Error; };
class ValidationError : public Error { using Error::Error; };

// Throws the qvsim error type matching a qvg status (include/qvg.h).
void check_status(int status);

// ---- gate library (reference gates.hpp:12-37, gates.cpp) ----------------------
inline constexpr double kBuiltinUnitaryTol = 1e-9;
inline constexpr double kCustomUnitaryTol = 1e-6;

// The reference library (h x y z s sdg t tdg rx ry rz u) plus the gates the
// BASELINE configs need and the reference lacks: p (phase,
// 1 angle), u3 (3 angles), sx sy sw (sqrt X/Y/W).
std::optional<std::size_t> gate_arity(const std::string &name);
const std::vector<std::string> &builtin_gate_names();
GateMatrix make_gate(const std::string &name, const std::vector<double> &params, bool strict = false);
GateOp single_op(const std::string &name, std::uint32_t target, std::vector<double> params = {});
// Reference: cx, cz (gates.cpp:95-107). Added: cp <theta> (controlled phase,
// R_k of the QFT) and cu <8 reals> (controlled arbitrary unitary).
GateOp controlled_op(const std::string &name, std::uint32_t control, std::uint32_t target,
                     std::vector<double> params = {});

// ---- circuit text (reference circuit_io.hpp:26-33) ----------------------------
Circuit parse_circuit(std::string_view text, std::optional<std::uint32_t> n_override = {}, bool strict = false);
std::string serialize_circuit(const Circuit &c);

// ---- seeded generators (reference engine.hpp:61-80, engine.cpp:159-251) ------
std::uint64_t uniform_below(std::mt19937_64 &rng, std::uint64_t bound);
double uniform_unit(std::mt19937_64 &rng);
Circuit random_circuit(std::uint32_t n_qubits, std::uint32_t depth, std::uint64_t seed);
Circuit random_circuit(std::mt19937_64 &rng, std::uint32_t n_qubits, std::uint32_t depth);
Circuit make_benchmark_circuit(std::uint32_t n_qubits);

// ---- BASELINE config circuits -------------------------------------
// C0 / C4: `layers` x (U3 on every qubit, then CX(q -> q+1) ladder).
Circuit u3_ladder_circuit(std::uint32_t n_qubits, std::uint32_t layers, std::uint64_t seed);
// C1: X on the bits of a seeded basis index b, H on all qubits, QFT
// (H + controlled-phase R_k, 2pi/2^k), bit-reversal SWAPs as 3 CX each.
// h_layer = false drops the H layer: the output is then the plain QFT of |b>,
// amplitude 2^(-n/2) e^(2 pi i b y / 2^n) at y (an analytic check at any n).
Circuit qft_circuit(std::uint32_t n_qubits, std::uint64_t seed, std::uint64_t *basis_index = nullptr,
                    bool h_layer = true);
// C2: one Haar-random U per qubit q = 0..n-1, then CX(c, t) for every ordered
// pair with |c - t| in {1, 15, 29}.
Circuit haar_sweep_circuit(std::uint32_t n_qubits, std::uint64_t seed);
// C3: rows x cols grid, `cycles` cycles of {sqrt X, sqrt Y, sqrt W} (never
// repeating a qubit's previous draw) then CZ on edge pattern (cycle mod 4).
Circuit grid_circuit(std::uint32_t rows, std::uint32_t cols, std::uint32_t cycles, std::uint64_t seed);

// Flatten to the C-ABI op array (reference GateOp -> qvg_gate).
std::vector<qvg_gate> to_gates(const Circuit &c);
Circuit from_gates(std::uint32_t n_qubits, const qvg_gate *ops, std::size_t count);

// ---- engine (reference engine.hpp:21-59, metrics.hpp:14-30) ------------------
enum class Strategy { dense, paired, paired_cached, paired_cached_parallel, gpu };
const char *strategy_tag(Strategy s);
std::optional<Strategy> parse_strategy(std::string_view tag);
const std::vector<std::string> &strategy_tags();

struct RunConfig {
    Strategy strategy = Strategy::gpu;
    bool fuse = true;               // fused tile passes (QVG_OPT_FUSE)
    std::uint32_t tile_qubits = 0;  // 0: engine default
    bool sync = true;               // wait for the device before returning
    // StateStore path: 0 = the whole state in HBM when it fits, else stream
    // the file through two HBM windows (out-of-core); > 0 forces streaming
    // with windows of 2^window_qubits amplitudes.
    std::uint32_t window_qubits = 0;
};

// The reference's Metrics (reference metrics.hpp:14-30, to_json
// metrics.cpp:25-41) plus the GPU pass accounting. Store fields count the QVSV
// file traffic of a StateStore run; cache_* stay 0 (no host window);
// peak_cache_bytes is the device memory holding the state (or the two
// streaming windows).
struct Metrics {
    std::uint64_t bytes_read = 0;     // state-file bytes read (StateStore path)
    std::uint64_t bytes_written = 0;  // state-file bytes written
    std::uint64_t blocks_read = 0;    // state-file blocks read
    std::uint64_t blocks_written = 0;
    std::uint64_t cache_hits = 0;
    std::uint64_t cache_misses = 0;
    std::uint64_t peak_cache_bytes = 0;
    std::uint64_t gates_applied = 0;
    std::uint64_t traversals = 0;  // HBM passes (the reference's one traversal per gate)
    std::uint64_t fused_passes = 0;
    std::uint64_t bytes_moved = 0;
    std::uint64_t exchange_bytes = 0;
    std::uint64_t exchanges = 0;
    double wall_ms = 0.0;
    std::uint32_t workers = 1;  // GPUs (shards)
    std::string strategy;
};

// Device-resident state vector: the HBM replacement for BlockStore
// (reference store.hpp:47-100). Move-only, owns its qvg_state.
class StateVector {
  public:
    static StateVector create(std::uint32_t n_qubits, std::uint32_t precision = 128, int device = 0);
    static StateVector create_sharded(std::uint32_t n_qubits, std::uint32_t precision, int device,
                                      std::uint32_t rank, std::uint32_t world, const void *nccl_id);
    StateVector(StateVector &&o) noexcept;
    StateVector &operator=(StateVector &&o) noexcept;
    StateVector(const StateVector &) = delete;
    StateVector &operator=(const StateVector &) = delete;
    ~StateVector();

    std::uint32_t n_qubits() const noexcept { return n_; }
    std::uint64_t n_amps() const noexcept { return std::uint64_t{1} << n_; }
    std::uint32_t precision() const noexcept { return precision_; }
    std::uint32_t rank() const noexcept { return rank_; }
    std::uint32_t world() const noexcept { return world_; }
    qvg_state *handle() const noexcept { return s_; }

    void init_basis(std::uint64_t index);
    // Amplitudes are complex128 on the host; complex64 states convert.
    void load(const amp_t *amps, std::uint64_t offset, std::uint64_t count);
    void read(amp_t *out, std::uint64_t offset, std::uint64_t count) const;
    amp_t amplitude(std::uint64_t index) const;
    double norm() const;
    void probabilities(double *out, std::uint64_t offset, std::uint64_t count) const;
    std::vector<std::pair<std::uint64_t, amp_t>> top_amplitudes(std::size_t k) const;
    void set_option(int key, std::int64_t value);
    qvg_stats stats() const;
    void sync() const;

  private:
    explicit StateVector(qvg_state *s);
    qvg_state *s_ = nullptr;
    std::uint32_t n_ = 0, precision_ = 128, rank_ = 0, world_ = 1;
};

// Reference apply_circuit (engine.cpp:86-157) for the device-resident state.
// Only Strategy::gpu runs here; the CPU strategies belong to the reference's
// block-store engine. Metrics accumulate; wall_ms is this call's elapsed time.
void apply_circuit(StateVector &state, const Circuit &circuit, const RunConfig &config, Metrics &metrics);

// ---- QVSV state file (the reference's on-disk format) ------------------------
// 32-byte header: "QVSV", u32 version 1, u32 n_qubits, u64 block_amps, 12 zero
// bytes; then 2^n complex128 little-endian, index-ascending (reference
// store.hpp:24-29, 47-57). Files are interchangeable with the reference's
// BlockStore; block_amps is kept for that compatibility (the GPU path moves
// the state in large pinned chunks, not blocks).
inline constexpr std::uint64_t kDefaultBlockAmps = 65536;
inline constexpr std::uint32_t kMaxQubits = 58;

class StateStore {
  public:
    // |0...0>: a sparse file with amplitude 0 = 1 (reference store.cpp:181-214).
    static StateStore create(const std::string &path, std::uint32_t n_qubits,
                             std::uint64_t block_amps = kDefaultBlockAmps, bool overwrite = false);
    static StateStore open(const std::string &path);
    StateStore(StateStore &&o) noexcept;
    StateStore &operator=(StateStore &&o) noexcept;
    StateStore(const StateStore &) = delete;
    StateStore &operator=(const StateStore &) = delete;
    ~StateStore();

    const std::string &path() const noexcept { return path_; }
    std::uint32_t n_qubits() const noexcept { return n_; }
    std::uint64_t n_amps() const noexcept { return std::uint64_t{1} << n_; }
    std::uint64_t block_amps() const noexcept { return block_amps_; }
    std::uint64_t n_blocks() const noexcept { return n_amps() / block_amps_; }

    void read(amp_t *out, std::uint64_t offset, std::uint64_t count) const;
    void write(const amp_t *in, std::uint64_t offset, std::uint64_t count);
    amp_t amplitude(std::uint64_t index) const;
    double norm() const;  // Kahan, like BlockStore::norm (store.cpp:301-316)
    void sync() const;

  private:
    StateStore(int fd, std::string path, std::uint32_t n, std::uint64_t block_amps);
    int fd_ = -1;
    std::string path_;
    std::uint32_t n_ = 0;
    std::uint64_t block_amps_ = 0;
};

// The drop-in for the reference's apply_circuit(BlockStore&, ...) with
// strategy "gpu": the file streams into HBM through pinned chunks, the circuit
// runs on the device, and the state streams back.
void apply_circuit(StateStore &store, const Circuit &circuit, const RunConfig &config, Metrics &metrics,
                   int device = 0);

// reference top_amplitudes (engine.cpp:511-544): k largest |a|^2, ties by index.
std::vector<std::pair<std::uint64_t, amp_t>> top_amplitudes(const StateStore &store, std::size_t k);

// reference verify_equivalence (engine.hpp:82-121, engine.cpp:253-340) for the
// GPU strategy. Each trial draws the reference's own random circuit (same
// per-trial seed derivation). Its reference run is one HBM pass per gate
// (the kernels that restate apply_pair). It is compared against every other
// device configuration: fused tiles (default and 5-qubit tiles), 2 and 4
// virtual shards, and the out-of-core window path. A failure records the
// first gate whose post-state already differs.
struct VerifyOptions {
    std::uint32_t min_qubits = 1;
    std::uint32_t max_qubits = 10;
    std::uint32_t max_depth = 30;
    std::uint64_t trials = 200;
    std::uint64_t seed = 1;
    double tolerance = 1e-12;
    int device = 0;
};

struct VerifyFailure {
    std::uint64_t trial = 0;
    std::uint32_t n_qubits = 0;
    std::uint32_t depth = 0;
    std::string config;
    double deviation = 0.0;
    std::optional<std::size_t> first_divergent_gate;
};

struct VerifyResult {
    std::uint64_t trials = 0;
    std::uint64_t comparisons = 0;
    double max_deviation = 0.0;
    std::vector<VerifyFailure> failures;
    bool passed() const noexcept { return failures.empty(); }
};

VerifyResult verify_equivalence(const VerifyOptions &opts);

}  // namespace qvsim
