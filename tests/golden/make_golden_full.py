"""Full-size golden fixtures for BASELINE configs 2 and 3 (n = 30, complex128),
generated ONCE in the build container by the UNMODIFIED reference engine
(oracle/_ref/libqvsim_ref.so, `make -C oracle ref`) and committed. TEST
INFRASTRUCTURE ONLY; the GPU box never runs this (it has no reference tree).

    nice python tests/golden/make_golden_full.py [config2|config3 ...]

For each config the reference's `apply_circuit` runs with
`paired-cached-parallel` (workers = all cores, 64 MiB window per worker,
65536-amplitude blocks, the QVSV store on /dev/shm — SURVEY §8d's CPU setup)
from |0...0>. The final QVSV payload is memory-mapped and summarised:

  chunk_sha256   sha256 of every 2^26-amplitude (1 GiB) chunk, in order
  norm           the reference's own Kahan norm (BlockStore::norm,
                 reference store.cpp:301-316)
  top8           the 8 largest |a|^2 (ties by lower index) with their values
  samples        1024 amplitudes at seeded indices (numpy default_rng(seed))
  ops_file       the exact qvg_gate records fed to the engine (.npy beside
                 this file); bench.py's reference arm loads config 2's
  provenance     builder + args, seed, sha256 of this script, of the
                 reference sources compiled, and the engine's wall time

The circuits are built by the package's host layer (the same builders the
GPU tests call); ops_sha256 pins those bytes, so the GPU tests check that
the builder still emits them.
"""
from __future__ import annotations

import glob
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import GATE_DTYPE, RefEngine  # noqa: E402

CHUNK = 1 << 26
N_SAMPLES = 1024
SAMPLE_SEED = 2508
FULL = {
    # name: (builder, args, ops file)
    "config2": ("config2_haar_sweep_n30", "haar_sweep_circuit", (30, 2508), "config2_haar_sweep_n30_ops.npy"),
    "config3": ("config3_grid_5x6_c24_n30", "grid_circuit", (5, 6, 24, 1), "config3_grid_5x6_c24_n30_ops.npy"),
}
OUT = os.path.join(HERE, "ref_full.json")


def sha(b) -> str:
    return hashlib.sha256(b).hexdigest()


def sample_indices(n: int) -> np.ndarray:
    return np.sort(np.random.default_rng(SAMPLE_SEED).choice(1 << n, N_SAMPLES, replace=False))


def top8(amps: np.ndarray) -> list[int]:
    """Indices of the 8 largest re*re + im*im, ties by lower index."""
    cand_i, cand_p = [], []
    for off in range(0, amps.size, CHUNK):
        c = np.asarray(amps[off:off + CHUNK])
        p = c.real * c.real + c.imag * c.imag
        k = min(8, p.size)
        thr = np.partition(p, p.size - k)[p.size - k]
        idx = np.nonzero(p >= thr)[0]
        cand_i.append(idx + off)
        cand_p.append(p[idx])
    i = np.concatenate(cand_i)
    p = np.concatenate(cand_p)
    order = np.lexsort((i, -p))
    return [int(x) for x in i[order[:8]]]


def ref_sources_sha() -> str:
    h = hashlib.sha256()
    for f in sorted(glob.glob("/root/reference/proj/src/*.cpp") + glob.glob("/root/reference/proj/include/qvsim/*.hpp")):
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def generate(key: str) -> dict:
    import paper_2508_15545_b200 as qv

    name, fn, args, ops_file = FULL[key]
    out = getattr(qv, fn)(*args)
    c = out[0] if isinstance(out, tuple) else out
    n = c.n_qubits
    ops = np.frombuffer(c.gates().tobytes(), dtype=GATE_DTYPE).copy()
    np.save(os.path.join(HERE, ops_file), ops)
    workers = os.cpu_count() or 1
    eng = RefEngine()
    t0 = time.time()
    with eng.store(n, block_amps=65536, scratch="/dev/shm") as st:
        wall_ms = st.apply(ops, "paired-cached-parallel", workers, workers * (64 << 20))
        st.sync()
        norm = st.norm()
        amps = st.amplitudes()
        chunks = [sha(np.asarray(amps[o:o + CHUNK]).tobytes()) for o in range(0, amps.size, CHUNK)]
        t8 = top8(amps)
        si = sample_indices(n)
        sv = np.asarray(amps[si])
        rec = {
            "builder": fn, "args": list(args), "n_qubits": n, "n_ops": int(len(ops)),
            "ops_file": ops_file, "ops_sha256": sha(ops.tobytes()),
            "chunk_amps": CHUNK, "chunk_sha256": chunks, "norm": norm,
            "top8_index": t8, "top8": [[float(amps[i].real), float(amps[i].imag)] for i in t8],
            "sample_seed": SAMPLE_SEED, "samples": [[float(a.real), float(a.imag)] for a in sv],
            "engine": f"reference apply_circuit paired-cached-parallel, workers={workers}, "
                      f"cache_bytes={workers}x64MiB, block_amps=65536, store on /dev/shm",
            "engine_wall_ms": wall_ms, "generated_s": round(time.time() - t0, 1),
            "generator_sha256": sha(open(os.path.abspath(__file__), "rb").read()),
            "reference_sources_sha256": ref_sources_sha(),
        }
        del amps
    return rec


def main(keys):
    fx = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            fx = json.load(f)
    for key in keys:
        rec = generate(key)
        fx[FULL[key][0]] = rec
        with open(OUT, "w") as f:
            json.dump(fx, f, indent=1)
        print(key, "done in", rec["generated_s"], "s; engine", rec["engine_wall_ms"] / 1e3, "s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(FULL))
