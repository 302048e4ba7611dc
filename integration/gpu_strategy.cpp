// gpu_strategy.cpp — the `Strategy::gpu` branch a maintainer adds to the
// reference engine, compiled against the reference's own
// headers and linked with libqvg.so by oracle/Makefile (`make -C oracle
// dropin`). The reference's binding then forwards strategy="gpu" unchanged
// (reference bindings/module.cpp:118-139 -> parse_strategy).
#include "qvsim/gpu_strategy.hpp"

#include <cstdint>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "qvg.h"
#include "qvsim/engine.hpp"
#include "qvsim/error.hpp"

namespace qvsim {
namespace {

void qvg_throw(int rc) {  // status -> reference error tree (error.hpp:10-50)
    if (rc == QVG_OK) return;
    const std::string msg = std::string("gpu strategy: ") + qvg_last_error();
    switch (rc) {
    case QVG_ERR_VALIDATION: throw ValidationError(msg);
    case QVG_ERR_CAPACITY: throw CapacityError(msg);
    case QVG_ERR_FORMAT: throw FormatError(msg);
    default: throw IoError(msg);  // CUDA / NCCL failure, no device
    }
}

qvg_gate flatten(const GateOp &op) {  // GateOp (types.hpp:43-52) -> qvg_gate
    qvg_gate g{};
    g.kind = op.kind == OpKind::controlled ? QVG_OP_CONTROLLED : QVG_OP_SINGLE;
    g.target = op.target;
    g.control = op.control ? static_cast<int32_t>(*op.control) : -1;
    const amp_t m[4] = {op.matrix.u00, op.matrix.u01, op.matrix.u10, op.matrix.u11};
    for (int i = 0; i < 4; ++i) {
        g.u[2 * i] = m[i].real();
        g.u[2 * i + 1] = m[i].imag();
    }
    return g;
}

}  // namespace

void apply_circuit_gpu(BlockStore &store, const Circuit &circuit, Metrics &metrics) {
    const char *dev_env = std::getenv("QVSIM_GPU_DEVICE");
    qvg_state *dev = nullptr;
    qvg_throw(qvg_create(store.n_qubits(), QVG_C128, dev_env ? std::atoi(dev_env) : 0, &dev));
    std::unique_ptr<qvg_state, int (*)(qvg_state *)> guard(dev, qvg_destroy);
    DenseState state = read_full_state(store, metrics);  // reference engine.cpp:483-494
    // amp_t is std::complex<double>: the interleaved complex128 layout qvg_load takes
    qvg_throw(qvg_load(dev, state.amps.data(), 0, state.amps.size()));
    std::vector<qvg_gate> gates;
    gates.reserve(circuit.ops.size());
    for (const GateOp &op : circuit.ops) gates.push_back(flatten(op));
    qvg_throw(qvg_apply(dev, gates.data(), gates.size()));
    qvg_throw(qvg_read(dev, state.amps.data(), 0, state.amps.size()));  // waits for the device
    write_full_state(store, state, metrics);  // reference engine.cpp:496-509
    qvg_stats st{};
    qvg_throw(qvg_stats_get(dev, &st));
    metrics.gates_applied += st.gates_applied;
    metrics.traversals += st.passes;  // HBM passes (fused tiles count once)
}

}  // namespace qvsim
