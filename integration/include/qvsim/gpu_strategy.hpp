// gpu_strategy.hpp — the reference-side drop-in: the
// declaration the patched reference engine.cpp includes for its new
// `case Strategy::gpu` branch (reference engine.cpp:109-150).
#pragma once

#include "qvsim/metrics.hpp"
#include "qvsim/store.hpp"
#include "qvsim/types.hpp"

namespace qvsim {

/// Strategy::gpu: read the store's state, apply the circuit on the B200
/// through libqvg.so (include/qvg.h), write the state back — the dense
/// strategy's read-full -> compute -> write-full shape (reference
/// engine.cpp:110-127). libqvg status codes map onto the reference's error
/// tree (error.hpp:10-50). Counters: gates_applied += ops, traversals +=
/// HBM passes.
void apply_circuit_gpu(BlockStore &store, const Circuit &circuit, Metrics &metrics);

}  // namespace qvsim
