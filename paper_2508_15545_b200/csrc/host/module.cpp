// module.cpp — pybind11 module `_core`: the Python face of the host layer,
// mirroring the reference's binding (reference proj/bindings/module.cpp:40-188)
// with StateVector (device-resident) in place of StateStore and
// strategy="gpu". Unlike the reference, the GIL is released while the device
// works.
#include <pybind11/complex.h>
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cstring>

#include "qvsim_gpu.hpp"

namespace py = pybind11;
using namespace qvsim;

namespace {

py::array_t<std::uint8_t> gates_bytes(const std::vector<qvg_gate> &g) {
    py::array_t<std::uint8_t> out(g.size() * sizeof(qvg_gate));
    if (!g.empty()) std::memcpy(out.mutable_data(), g.data(), g.size() * sizeof(qvg_gate));
    return out;
}

const qvg_gate *gate_ptr(const py::buffer_info &b, std::size_t &count) {
    const std::size_t bytes = (std::size_t)(b.size * b.itemsize);
    if (bytes % sizeof(qvg_gate)) throw ValidationError("gate buffer is not a whole number of 80-byte qvg_gate records");
    count = bytes / sizeof(qvg_gate);
    return static_cast<const qvg_gate *>(b.ptr);
}

py::dict metrics_dict(const Metrics &m, std::uint32_t n) {
    py::dict d;
    d["n_qubits"] = n;
    d["strategy"] = m.strategy;
    d["workers"] = m.workers;
    d["gates_applied"] = m.gates_applied;
    d["traversals"] = m.traversals;
    d["blocks_read"] = m.blocks_read;
    d["blocks_written"] = m.blocks_written;
    d["bytes_read"] = m.bytes_read;
    d["bytes_written"] = m.bytes_written;
    d["cache_hits"] = m.cache_hits;
    d["cache_misses"] = m.cache_misses;
    d["peak_cache_bytes"] = m.peak_cache_bytes;
    d["fused_passes"] = m.fused_passes;
    d["bytes_moved"] = m.bytes_moved;
    d["exchange_bytes"] = m.exchange_bytes;
    d["exchanges"] = m.exchanges;
    d["wall_ms"] = m.wall_ms;
    return d;
}

py::dict stats_dict(const qvg_stats &s) {
    py::dict d;
    d["gates_applied"] = s.gates_applied;
    d["passes"] = s.passes;
    d["fused_passes"] = s.fused_passes;
    d["kernel_launches"] = s.kernel_launches;
    d["bytes_moved"] = s.bytes_moved;
    d["exchange_bytes"] = s.exchange_bytes;
    d["exchanges"] = s.exchanges;
    d["kernel_ms"] = s.kernel_ms;
    d["exchange_ms"] = s.exchange_ms;
    d["fused_exchanges"] = s.fused_exchanges;
    d["graph_replays"] = s.graph_replays;
    d["jit_passes"] = s.jit_passes;
    return d;
}

}  // namespace

PYBIND11_MODULE(_core, m) {
    m.doc() = "B200-native gate application for the QVecOpt state-vector simulator";

    auto base = py::register_exception<Error>(m, "QvsimError");
    py::register_exception<ValidationError>(m, "ValidationError", base.ptr());
    py::register_exception<CapacityError>(m, "CapacityError", base.ptr());
    py::register_exception<IoError>(m, "IoError", base.ptr());
    py::register_exception<FormatError>(m, "FormatError", base.ptr());
    py::register_exception<ParseError>(m, "ParseError", base.ptr());

    py::class_<Circuit>(m, "Circuit", "Ordered gate list on n qubits")
        .def_property_readonly("n_qubits", [](const Circuit &c) { return c.n_qubits; })
        .def("__len__", [](const Circuit &c) { return c.ops.size(); })
        .def("to_text", &serialize_circuit, "Circuit text that parse_circuit round-trips exactly")
        .def("gates", [](const Circuit &c) { return gates_bytes(to_gates(c)); },
             "The ops as packed qvg_gate records (80 bytes each, include/qvg.h)")
        .def("names", [](const Circuit &c) {
            std::vector<std::string> out;
            for (const auto &op : c.ops) out.push_back(op.name);
            return out;
        })
        .def("__repr__", [](const Circuit &c) {
            return "<Circuit n_qubits=" + std::to_string(c.n_qubits) + " ops=" + std::to_string(c.ops.size()) + ">";
        });

    m.def("circuit_from_gates", [](std::uint32_t n, py::buffer buf) {
        const py::buffer_info b = buf.request();
        std::size_t count = 0;
        const qvg_gate *g = gate_ptr(b, count);
        return from_gates(n, g, count);
    }, py::arg("n_qubits"), py::arg("gates"));

    m.def("parse_circuit",
          [](const std::string &text, std::optional<std::uint32_t> qubits, bool strict) {
              return parse_circuit(text, qubits, strict);
          },
          py::arg("text"), py::arg("qubits") = std::nullopt, py::arg("strict") = false);
    m.def("serialize_circuit", &serialize_circuit, py::arg("circuit"));
    m.def("random_circuit",
          [](std::uint32_t n, std::uint32_t depth, std::uint64_t seed) { return random_circuit(n, depth, seed); },
          py::arg("n_qubits"), py::arg("depth"), py::arg("seed"));
    m.def("make_benchmark_circuit", &make_benchmark_circuit, py::arg("n_qubits"));
    m.def("u3_ladder_circuit", &u3_ladder_circuit, py::arg("n_qubits"), py::arg("layers") = 20, py::arg("seed") = 1);
    m.def("qft_circuit", [](std::uint32_t n, std::uint64_t seed, bool h_layer) {
        std::uint64_t b = 0;
        Circuit c = qft_circuit(n, seed, &b, h_layer);
        return py::make_tuple(c, b);
    }, py::arg("n_qubits"), py::arg("seed") = 1, py::arg("h_layer") = true, "(circuit, basis index b)");
    m.def("haar_sweep_circuit", &haar_sweep_circuit, py::arg("n_qubits"), py::arg("seed") = 1);
    m.def("grid_circuit", &grid_circuit, py::arg("rows") = 5, py::arg("cols") = 6, py::arg("cycles") = 24,
          py::arg("seed") = 1);
    m.def("make_gate", [](const std::string &name, const std::vector<double> &p, bool strict) {
        const GateMatrix g = make_gate(name, p, strict);
        return std::vector<amp_t>{g.u00, g.u01, g.u10, g.u11};
    }, py::arg("name"), py::arg("params") = std::vector<double>{}, py::arg("strict") = false);
    m.def("strategy_tags", &strategy_tags);

    py::class_<StateVector>(m, "StateVector", "Device-resident state vector (HBM), the GPU analog of StateStore")
        .def_static("create", &StateVector::create, py::arg("n_qubits"), py::arg("precision") = 128,
                    py::arg("device") = 0, "New state holding |0...0>")
        .def_static("create_sharded",
                    [](std::uint32_t n, std::uint32_t precision, int device, std::uint32_t rank, std::uint32_t world,
                       std::optional<py::bytes> nccl_id) {
                        if (!nccl_id)
                            return StateVector::create_sharded(n, precision, device, rank, world, nullptr);
                        const std::string id = *nccl_id;
                        if (id.size() != 128) throw ValidationError("nccl_id must be 128 bytes");
                        py::gil_scoped_release nogil;
                        return StateVector::create_sharded(n, precision, device, rank, world, id.data());
                    },
                    py::arg("n_qubits"), py::arg("precision"), py::arg("device"), py::arg("rank"), py::arg("world"),
                    py::arg("nccl_id") = std::nullopt,
                    "Sharded state; nccl_id=None keeps all shards on this device (virtual shards)")
        .def_property_readonly("n_qubits", &StateVector::n_qubits)
        .def_property_readonly("n_amps", &StateVector::n_amps)
        .def_property_readonly("precision", &StateVector::precision)
        .def_property_readonly("rank", &StateVector::rank)
        .def_property_readonly("world", &StateVector::world)
        .def("init_basis", &StateVector::init_basis, py::arg("index"))
        .def("norm", [](const StateVector &s) {
            py::gil_scoped_release nogil;
            return s.norm();
        })
        .def("amplitude", &StateVector::amplitude, py::arg("index"))
        .def("read_state", [](const StateVector &s, std::uint64_t offset, std::optional<std::uint64_t> count) {
            const std::uint64_t c = count ? *count : s.n_amps() - std::min(offset, s.n_amps());
            py::array_t<std::complex<double>> out(c);
            {
                py::gil_scoped_release nogil;
                s.read(out.mutable_data(), offset, c);
            }
            return out;
        }, py::arg("offset") = 0, py::arg("count") = std::nullopt, "Amplitudes as a complex128 numpy array")
        .def("load_async", [](StateVector &s, py::buffer buf, std::uint64_t offset) {
            const py::buffer_info b = buf.request();
            const std::size_t amp = s.precision() == 128 ? 16 : 8;
            if ((std::size_t)(b.size * b.itemsize) % amp) throw ValidationError("buffer is not whole amplitudes");
            check_status(qvg_load_async(s.handle(), b.ptr, offset, (std::uint64_t)(b.size * b.itemsize) / amp));
        }, py::arg("amps"), py::arg("offset") = 0,
           "Stream-ordered H2D in the state's precision; keep the (pinned) buffer alive until sync()")
        .def("read_async", [](StateVector &s, py::buffer buf, std::uint64_t offset) {
            const py::buffer_info b = buf.request(true);
            const std::size_t amp = s.precision() == 128 ? 16 : 8;
            if ((std::size_t)(b.size * b.itemsize) % amp) throw ValidationError("buffer is not whole amplitudes");
            check_status(qvg_read_async(s.handle(), b.ptr, offset, (std::uint64_t)(b.size * b.itemsize) / amp));
        }, py::arg("out"), py::arg("offset") = 0,
           "Stream-ordered D2H in the state's precision; the data is valid after sync()")
        .def("read_into",[](const StateVector &s, py::array_t<std::complex<double>, py::array::c_style> out,
                             std::uint64_t offset) {
            const std::uint64_t c = (std::uint64_t)out.size();
            amp_t *p = out.mutable_data();
            py::gil_scoped_release nogil;
            s.read(p, offset, c);
        }, py::arg("out"), py::arg("offset") = 0, "Amplitudes into a caller-owned (e.g. pinned) complex128 array")
        .def("load_state", [](StateVector &s,py::array_t<std::complex<double>, py::array::c_style | py::array::forcecast> a,
                              std::uint64_t offset) {
            const std::uint64_t c = (std::uint64_t)a.size();
            const amp_t *p = a.data();
            py::gil_scoped_release nogil;
            s.load(p, offset, c);
        }, py::arg("amps"), py::arg("offset") = 0)
        .def("probabilities", [](const StateVector &s, std::uint64_t offset, std::optional<std::uint64_t> count) {
            const std::uint64_t c = count ? *count : s.n_amps() - std::min(offset, s.n_amps());
            py::array_t<double> out(c);
            {
                py::gil_scoped_release nogil;
                s.probabilities(out.mutable_data(), offset, c);
            }
            return out;
        }, py::arg("offset") = 0, py::arg("count") = std::nullopt)
        .def("top_amplitudes", [](const StateVector &s, std::size_t k) {
            py::gil_scoped_release nogil;
            return s.top_amplitudes(k);
        }, py::arg("k") = 8)
        .def("inner", [](StateVector &a, StateVector &b) {
            double re = 0, im = 0;
            {
                py::gil_scoped_release nogil;
                check_status(qvg_inner_product(a.handle(), b.handle(), &re, &im));
            }
            return std::complex<double>(re, im);
        }, py::arg("other"), "<self|other> = sum conj(a_i) b_i on the device")
        .def("fidelity", [](StateVector &a, StateVector &b) {
            double re = 0, im = 0;
            {
                py::gil_scoped_release nogil;
                check_status(qvg_inner_product(a.handle(), b.handle(), &re, &im));
            }
            return re * re + im * im;
        }, py::arg("other"), "|<self|other>|^2")
        .def("max_deviation", [](StateVector &a, StateVector &b) {
            double m = 0;
            {
                py::gil_scoped_release nogil;
                check_status(qvg_max_deviation(a.handle(), b.handle(), &m));
            }
            return m;
        }, py::arg("other"), "max_i |a_i - b_i| on the device")
        .def("set_option", &StateVector::set_option, py::arg("key"), py::arg("value"))
        .def("stats", [](const StateVector &s) { return stats_dict(s.stats()); })
        .def("checksums",
             [](StateVector &s, std::uint64_t chunk_amps) {
                 std::uint64_t n = 0;
                 check_status(qvg_checksums(s.handle(), chunk_amps, nullptr, 0, &n));
                 py::array_t<std::uint64_t> out({(py::ssize_t)n, (py::ssize_t)2});
                 {
                     py::gil_scoped_release nogil;
                     check_status(qvg_checksums(s.handle(), chunk_amps, out.mutable_data(), n, &n));
                 }
                 return out;
             },
             py::arg("chunk_amps") = std::uint64_t{1} << 26,
             "(chunks, 2) uint64 checksum words of the state in canonical order (qvg_checksums)")
        .def("handle", [](const StateVector &s) { return reinterpret_cast<std::uintptr_t>(s.handle()); },
             "the qvg_state* of this state (for C-ABI calls through ctypes, e.g. qvg_set_step_hook)")
        .def("reset_stats", [](StateVector &s) { check_status(qvg_stats_reset(s.handle())); })
        .def("sync", [](const StateVector &s) {
            py::gil_scoped_release nogil;
            s.sync();
        })
        .def("stream", [](const StateVector &s) {
            void *st = nullptr;
            check_status(qvg_stream(s.handle(), &st));
            return (std::uintptr_t)st;
        }, "cudaStream_t of the state's work, as an integer")
        .def("device_buffer", [](const StateVector &s) {
            void *p = nullptr;
            std::uint64_t bytes = 0;
            check_status(qvg_device_buffer(s.handle(), &p, &bytes));
            return py::make_tuple((std::uintptr_t)p, bytes);
        })
        .def("apply_gates", [](StateVector &s, py::buffer buf, bool sync) {
            const py::buffer_info b = buf.request();
            std::size_t count = 0;
            const qvg_gate *g = gate_ptr(b, count);
            py::gil_scoped_release nogil;
            check_status(qvg_apply(s.handle(), g, count));
            if (sync) s.sync();
        }, py::arg("gates"), py::arg("sync") = true, "Apply packed qvg_gate records (the C-ABI hot path)");

    m.def("apply_circuit",
          [](StateVector &state, const Circuit &circuit, const std::string &strategy, bool fuse,
             std::uint32_t tile_qubits, bool sync) {
              const auto s = parse_strategy(strategy);
              if (!s) throw ValidationError("unknown strategy '" + strategy + "'");
              RunConfig cfg;
              cfg.strategy = *s;
              cfg.fuse = fuse;
              cfg.tile_qubits = tile_qubits;
              cfg.sync = sync;
              Metrics metrics;
              {
                  py::gil_scoped_release nogil;
                  apply_circuit(state, circuit, cfg, metrics);
              }
              return metrics_dict(metrics, state.n_qubits());
          },
          py::arg("state"), py::arg("circuit"), py::arg("strategy") = "gpu", py::arg("fuse") = true,
          py::arg("tile_qubits") = 0, py::arg("sync") = true,
          "Apply the circuit in place on the device; returns the run's metrics document");

    py::class_<StateStore>(m, "StateStore", "QVSV state file, interchangeable with the reference's BlockStore")
        .def_static("create", [](const std::string &path, std::uint32_t n, std::uint64_t block_amps, bool overwrite) {
            const std::uint64_t ba = std::min<std::uint64_t>(block_amps, std::uint64_t{1} << std::min(n, 62u));
            return StateStore::create(path, n, ba, overwrite);
        }, py::arg("path"), py::arg("n_qubits"), py::arg("block_amps") = kDefaultBlockAmps,
           py::arg("overwrite") = false, "New store holding |0...0>; block_amps is capped at 2^n")
        .def_static("open", &StateStore::open, py::arg("path"))
        .def_property_readonly("n_qubits", &StateStore::n_qubits)
        .def_property_readonly("n_amps", &StateStore::n_amps)
        .def_property_readonly("block_amps", &StateStore::block_amps)
        .def_property_readonly("n_blocks", &StateStore::n_blocks)
        .def_property_readonly("path", &StateStore::path)
        .def("norm", &StateStore::norm)
        .def("amplitude", &StateStore::amplitude, py::arg("index"))
        .def("read_state", [](const StateStore &s) {
            py::array_t<std::complex<double>> out(s.n_amps());
            s.read(out.mutable_data(), 0, s.n_amps());
            return out;
        }, "All 2^n amplitudes (numpy complex128)")
        .def("sync", &StateStore::sync);

    m.def("apply_circuit",
          [](StateStore &store, const Circuit &circuit, const std::string &strategy, std::uint64_t cache_bytes,
             std::uint32_t workers, bool fuse, int device, std::uint32_t window_qubits) {
              const auto s = parse_strategy(strategy);
              if (!s) throw ValidationError("unknown strategy '" + strategy + "'");
              // cache_bytes / workers: the reference's positional signature
              // (reference bindings/module.cpp:118-139); the GPU strategy sizes
              // its HBM windows itself and has no host worker pool.
              if (workers == 0) throw ValidationError("workers must be >= 1");
              (void)cache_bytes;
              RunConfig cfg;
              cfg.strategy = *s;
              cfg.fuse = fuse;
              cfg.window_qubits = window_qubits;
              Metrics metrics;
              {
                  py::gil_scoped_release nogil;
                  apply_circuit(store, circuit, cfg, metrics, device);
              }
              py::dict d = metrics_dict(metrics, store.n_qubits());
              d["bytes_read"] = metrics.bytes_read;
              d["bytes_written"] = metrics.bytes_written;
              return d;
          },
          py::arg("store"), py::arg("circuit"), py::arg("strategy") = "gpu",
          py::arg("cache_bytes") = std::uint64_t{64} << 20, py::arg("workers") = 1, py::arg("fuse") = true,
          py::arg("device") = 0, py::arg("window_qubits") = 0,
          "File-backed apply: store -> HBM -> circuit on the GPU -> store; window_qubits > 0 (or a state larger "
          "than device memory) streams the file through two HBM windows instead");

    m.def("verify_equivalence",
          [](std::uint32_t max_qubits, std::uint64_t trials, std::uint32_t max_depth, std::uint64_t seed,
             const std::string &scratch_dir, int device) {
              (void)scratch_dir;  // the reference's store directory; device runs need none
              VerifyOptions opts;
              opts.max_qubits = max_qubits;
              opts.trials = trials;
              opts.max_depth = max_depth;
              opts.seed = seed;
              opts.device = device;
              VerifyResult r;
              {
                  py::gil_scoped_release nogil;
                  r = verify_equivalence(opts);
              }
              py::dict d;
              d["trials"] = r.trials;
              d["comparisons"] = r.comparisons;
              d["max_deviation"] = r.max_deviation;
              d["failures"] = r.failures.size();
              d["passed"] = r.passed();
              py::list details;
              for (const VerifyFailure &f : r.failures) {
                  py::dict e;
                  e["trial"] = f.trial;
                  e["n_qubits"] = f.n_qubits;
                  e["depth"] = f.depth;
                  e["config"] = f.config;
                  e["deviation"] = f.deviation;
                  if (f.first_divergent_gate) e["first_divergent_gate"] = *f.first_divergent_gate;
                  else e["first_divergent_gate"] = py::none();
                  details.append(e);
              }
              d["failure_details"] = details;
              return d;
          },
          py::arg("max_qubits") = 10, py::arg("trials") = 200, py::arg("max_depth") = 30, py::arg("seed") = 1,
          py::arg("scratch_dir") = "", py::arg("device") = 0,
          "Random circuits (the reference's verify_equivalence draws) through every device configuration, "
          "each compared with the one-pass-per-gate run");

    m.def("apply_circuit_host",
          [](py::buffer amps, const Circuit &circuit, std::uint32_t window_qubits, int device) {
              const py::buffer_info b = amps.request(true);
              const std::size_t bytes = (std::size_t)(b.size * b.itemsize);
              std::uint32_t precision = 0;
              if (b.format == py::format_descriptor<std::complex<double>>::format()) precision = 128;
              else if (b.format == py::format_descriptor<std::complex<float>>::format()) precision = 64;
              else throw ValidationError("amplitudes must be complex128 or complex64");
              const std::size_t count = bytes / (precision / 8);
              std::uint32_t n = 0;
              while ((std::size_t{1} << n) < count) ++n;
              if ((std::size_t{1} << n) != count) throw ValidationError("amplitude count is not a power of two");
              if (n != circuit.n_qubits) throw ValidationError("circuit qubit count does not match the state");
              const std::vector<qvg_gate> gates = to_gates(circuit);
              qvg_stats st{};
              {
                  py::gil_scoped_release nogil;
                  check_status(qvg_apply_host(b.ptr, n, precision, device, window_qubits, gates.data(), gates.size(),
                                              &st));
              }
              py::dict d = stats_dict(st);
              d["segments"] = st.exchanges;
              d["host_bytes"] = st.exchange_bytes;
              return d;
          },
          py::arg("amps"), py::arg("circuit"), py::arg("window_qubits"), py::arg("device") = 0,
          "Out-of-core apply: host-resident state streamed through a 2^window_qubits HBM window");

    m.def("top_amplitudes", [](const StateStore &store, std::size_t k) { return top_amplitudes(store, k); },
          py::arg("store"), py::arg("k") = 8, "(index, amplitude) pairs, largest magnitude first");
    m.def("top_amplitudes", [](const StateVector &state, std::size_t k) {
        py::gil_scoped_release nogil;
        return state.top_amplitudes(k);
    }, py::arg("store"), py::arg("k") = 8);
    m.attr("DEFAULT_BLOCK_AMPS") = kDefaultBlockAmps;

    m.def("nccl_unique_id", []() {
        std::string id(128, '\0');
        check_status(qvg_nccl_unique_id(id.data()));
        return py::bytes(id);
    });

    m.def("jit_info",
          [](bool) {
              std::uint64_t compiled = 0, failed = 0;
              double ms = 0;
              int avail = 0;
              check_status(qvg_jit_info(&compiled, &failed, &ms, &avail));
              py::dict d;
              d["compiled"] = compiled;
              d["failed"] = failed;
              d["compile_ms"] = ms;
              d["available"] = avail != 0;
              return d;
          },
          py::arg("drain") = false,
          "JIT tile-pass counters (process-wide): kernels compiled / failed, summed compile ms, NVRTC "
          "available (compiles finish inside the apply that needs them; `drain` is accepted and ignored)");
    m.def("jit_check",
          [](std::uint32_t n, py::buffer buf, std::uint32_t precision) {
              const py::buffer_info b = buf.request();
              std::size_t count = 0;
              const qvg_gate *g = gate_ptr(b, count);
              std::uint64_t passes = 0, compiled = 0;
              std::string err(4096, '\0');
              {
                  py::gil_scoped_release nogil;
                  check_status(qvg_jit_check(n, precision, g, count, &passes, &compiled, &err[0], err.size()));
              }
              err.resize(std::strlen(err.c_str()));
              return py::make_tuple(passes, compiled, err);
          },
          py::arg("n_qubits"), py::arg("gates"), py::arg("precision") = 128,
          "(fused passes, compiled, first error): generate and NVRTC-compile every fused pass's "
          "JIT-specialised kernel (host-only, no GPU)");

    m.def("plan_passes",
          [](std::uint32_t n, py::buffer buf, std::uint32_t precision, bool fuse, std::uint32_t tile_qubits,
             std::uint32_t carriers) {
              const py::buffer_info b = buf.request();
              std::size_t count = 0;
              const qvg_gate *g = gate_ptr(b, count);
              std::uint64_t passes = 0, fused = 0, bytes = 0;
              check_status(qvg_plan_passes(n, precision, fuse, tile_qubits, carriers, g, count, &passes, &fused, &bytes));
              return py::make_tuple(passes, fused, bytes);
          },
          py::arg("n_qubits"), py::arg("gates"), py::arg("precision") = 128, py::arg("fuse") = true,
          py::arg("tile_qubits") = 0, py::arg("carriers") = 0,
          "(passes, fused passes, algorithmic bytes) as qvg_apply plans them on an unsharded state "
          "(tile_qubits / carriers 0 = the engine's defaults for the precision and width)");

    m.def("shard_schedule",
          [](std::uint32_t n, std::uint32_t world, py::buffer buf, bool canonicalize, std::uint32_t batch) {
              const py::buffer_info b = buf.request();
              std::size_t count = 0;
              const qvg_gate *g = gate_ptr(b, count);
              std::uint64_t nsteps = 0;
              if (batch > 4) throw ValidationError("batch must be 0..4");
              const int flags = (canonicalize ? 1 : 0) | (int)(batch << 8);
              check_status(qvg_shard_schedule(n, world, g, count, flags, nullptr, 0, &nsteps));
              py::array_t<std::uint8_t> out(nsteps * sizeof(qvg_shard_step));
              check_status(qvg_shard_schedule(n, world, g, count, flags,
                                              reinterpret_cast<qvg_shard_step *>(out.mutable_data()), nsteps, &nsteps));
              return out;
          },
          py::arg("n_qubits"), py::arg("world"), py::arg("gates"), py::arg("canonicalize") = true,
          py::arg("batch") = 1,
          "Packed qvg_shard_step records (104 bytes each); batch = most global qubits one exchange swaps "
          "(the engine's default is 4)");

    m.attr("QVG_ABI_VERSION") = qvg_abi_version();
    m.attr("OPT_FUSE") = (int)QVG_OPT_FUSE;
    m.attr("OPT_TILE_QUBITS") = (int)QVG_OPT_TILE_QUBITS;
    m.attr("OPT_CARRIERS") = (int)QVG_OPT_CARRIERS;
    m.attr("OPT_LOW_KERNEL") = (int)QVG_OPT_LOW_KERNEL;
    m.attr("OPT_MIN_RUN") = (int)QVG_OPT_MIN_RUN;
    m.attr("OPT_PRED_STORE") = (int)QVG_OPT_PRED_STORE;
    m.attr("OPT_SUB_BITS") = (int)QVG_OPT_SUB_BITS;
    m.attr("OPT_FMA") = (int)QVG_OPT_FMA;
    m.attr("OPT_TIMING") = (int)QVG_OPT_TIMING;
    m.attr("OPT_EXCHANGE") = (int)QVG_OPT_EXCHANGE;
    m.attr("OPT_PREFETCH") = (int)QVG_OPT_PREFETCH;
    m.attr("OPT_BATCH_EXCHANGE") = (int)QVG_OPT_BATCH_EXCHANGE;
    m.attr("OPT_STAGE") = (int)QVG_OPT_STAGE;
    m.attr("OPT_GRAPH") = (int)QVG_OPT_GRAPH;
    m.attr("OPT_REORDER") = (int)QVG_OPT_REORDER;
    m.attr("OPT_CLASSES") = (int)QVG_OPT_CLASSES;
    m.attr("OPT_XCHG_CHUNK") = (int)QVG_OPT_XCHG_CHUNK;
    m.attr("OPT_PIPE") = (int)QVG_OPT_PIPE;
    m.attr("OPT_JIT") = (int)QVG_OPT_JIT;
    m.attr("OPT_PERM") = (int)QVG_OPT_PERM;
    m.attr("OPT_TILE_ORDER") = (int)QVG_OPT_TILE_ORDER;
    m.attr("OPT_TILE_GRID") = (int)QVG_OPT_TILE_GRID;
}
