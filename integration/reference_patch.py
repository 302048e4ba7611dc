"""Apply the `Strategy::gpu` branch to COPIES of the
reference's engine.hpp / engine.cpp. Build-time only: reads the reference
where it lies (default /root/reference/proj), writes the patched copies into a
git-ignored build directory (oracle/_ref/dropin by oracle/Makefile). Nothing
of the reference is committed here; the edits are anchored on the
reference's own lines and fail loudly if an anchor is missing.

    python integration/reference_patch.py <reference proj dir> <out dir>

Edits (reference line numbers as of the surveyed tree):
  include/qvsim/engine.hpp:21-33  enum class Strategy gains `gpu`
  src/engine.cpp:20-54            strategy_tag / parse_strategy / strategy_tags
                                  learn the tag "gpu"
  src/engine.cpp:109-150          apply_circuit's switch gains
                                  `case Strategy::gpu: apply_circuit_gpu(...)`
                                  (integration/gpu_strategy.cpp, libqvg.so)
"""
import os
import sys


def edit(text, anchor, new, where="after", count=1):
    if text.count(anchor) != count:
        raise SystemExit(f"reference_patch: anchor found {text.count(anchor)} times, expected {count}: {anchor!r}")
    i = text.index(anchor)
    if where == "after":
        i += len(anchor)
    return text[:i] + new + text[i:]


def main(ref, out):
    hpp = open(os.path.join(ref, "include", "qvsim", "engine.hpp")).read()
    hpp = edit(hpp, "    paired_cached_parallel,\n",
               "    /// libqvg.so (this repo): state copied into B200 HBM, the circuit\n"
               "    /// applied by the sm_100a kernels, the state written back.\n"
               "    gpu,\n")
    cpp = open(os.path.join(ref, "src", "engine.cpp")).read()
    cpp = edit(cpp, '#include "qvsim/engine.hpp"\n', '#include "qvsim/gpu_strategy.hpp"\n')
    cpp = edit(cpp, '        return "paired-cached-parallel";\n', '    case Strategy::gpu:\n        return "gpu";\n')
    cpp = edit(cpp, "    return std::nullopt;\n", '    if (tag == "gpu") {\n        return Strategy::gpu;\n    }\n',
               where="before")
    cpp = edit(cpp, '"dense", "paired", "paired-cached", "paired-cached-parallel"', ', "gpu"')
    cpp = edit(cpp, "                                   config.cache_bytes, metrics, config.hooks);\n            break;\n",
               "        case Strategy::gpu:\n            apply_circuit_gpu(store, circuit, metrics);\n            break;\n")
    os.makedirs(os.path.join(out, "include", "qvsim"), exist_ok=True)
    os.makedirs(os.path.join(out, "src"), exist_ok=True)
    with open(os.path.join(out, "include", "qvsim", "engine.hpp"), "w") as f:
        f.write(hpp)
    with open(os.path.join(out, "src", "engine.cpp"), "w") as f:
        f.write(cpp)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
