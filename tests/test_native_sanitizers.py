"""Host-side planning logic under AddressSanitizer + UndefinedBehaviorSanitizer
(SURVEY §5 "race detection / sanitizers": the reference has none).
tests/native/host_fuzz.cu drives make_plan, reorder_for_tiles, schedule_ops and
schedule_canonicalize over random op lists, options and shard counts, and
checks their invariants. It needs no GPU."""
import os
import shutil
import subprocess

import pytest

from conftest import ROOT

NVCC = "/usr/local/cuda/bin/nvcc"


@pytest.mark.skipif(not (os.path.exists(NVCC) and shutil.which("g++")), reason="needs nvcc and g++")
def test_host_planner_under_asan_ubsan(tmp_path):
    src = os.path.join(ROOT, "tests", "native", "host_fuzz.cu")
    obj, exe = str(tmp_path / "host_fuzz.o"), str(tmp_path / "host_fuzz")
    san = ["-Xcompiler", "-fsanitize=address", "-Xcompiler", "-fsanitize=undefined",
           "-Xcompiler", "-fno-omit-frame-pointer"]
    subprocess.run([NVCC, "-std=c++17", "-g", "-O1", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(ROOT, "paper_2508_15545_b200", "csrc"),
                    *san, "-c", "-o", obj, src], check=True, capture_output=True)
    subprocess.run(["g++", "-fsanitize=address", "-fsanitize=undefined", "-o", exe, obj,
                    "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"], check=True)
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=1",
               UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1")
    r = subprocess.run([exe, "1500"], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
    assert "runtime error" not in r.stderr
