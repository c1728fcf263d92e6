"""Host half of the library under AddressSanitizer + UndefinedBehaviorSanitizer (SURVEY §8 acceptance 3;
compute-sanitizer is closed on this GPU pool, so memory safety of the host code is checked here, on
CPU): the decomposer (both bands, level cap with residual), decomposition save/load incl. a corrupted
file, the distributed schedule for 2/4/8 ranks, and plan creation up to the missing device.  The
.cpp sources are recompiled with -fsanitize=address,undefined and linked with the library's nvcc
device objects into tests/sanitize/sanitize_main."""
import os
import shutil
import subprocess

import numpy as np
import pytest

import datagen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2402_19364_b200", "csrc")
BUILD = os.path.join(ROOT, "build", "sanitize")


def _build():
    from paper_2402_19364_b200 import build as b
    b.build()  # nvcc objects of the kernels (build/arrow_b200/*.cu.o)
    os.makedirs(BUILD, exist_ok=True)
    exe = os.path.join(BUILD, "sanitize_main")
    srcs = [os.path.join(CSRC, f) for f in ("decompose.cpp", "arrow_api.cpp", "dist.cpp", "comm.cpp", "layout.cpp")]
    srcs.append(os.path.join(ROOT, "tests", "sanitize", "sanitize_main.cpp"))
    objs = [os.path.join(ROOT, "build", "arrow_b200", f + ".o") for f in ("seg_kernel.cu", "kernels.cu", "gdecompose.cu")]
    inc_nccl, lib_nccl = b.nccl_paths()
    cuda = b.CUDA
    cmd = ["g++", "-std=c++17", "-O1", "-g", "-fno-omit-frame-pointer", "-fsanitize=address,undefined",
           "-fno-sanitize-recover=undefined", "-fopenmp", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           "-I", os.path.join(cuda, "include"), "-I", inc_nccl, *srcs, *objs, "-o", exe,
           "-L", os.path.join(cuda, "lib64"), "-lcudart", "-L", lib_nccl, "-l:libnccl.so.2",
           f"-Wl,-rpath,{lib_nccl}", f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    return exe


def _write_csr(path, g):
    with open(path, "wb") as f:
        f.write(np.int64(g.n).tobytes())
        f.write(np.int64(g.nnz).tobytes())
        f.write(g.row_ptr.astype("<i8").tobytes())
        f.write(g.col.astype("<i4").tobytes())
        f.write(np.asarray(g.val, dtype="<f8").tobytes())


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_host_half_under_asan_ubsan(tmp_path):
    exe = _build()
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=0:protect_shadow_gap=0",
               UBSAN_OPTIONS="print_stacktrace=1", CUDA_VISIBLE_DEVICES="")
    for spec, b in (("RMAT(12,4,1)", 256), ("GRID(64,1)", 64), ("PATH(500,3)", 3), ("TREE(2000,2)", 16),
                    ("RMAT(14,8,2)", 512)):
        g = datagen.make_graph(spec)
        path = str(tmp_path / "a.csr")
        _write_csr(path, g)
        r = subprocess.run([exe, path, str(b), str(tmp_path)], capture_output=True, text=True, env=env, timeout=600)
        out = r.stdout + r.stderr
        assert r.returncode == 0 and "SANITIZE_OK" in out, f"{spec}: {out[-4000:]}"
        assert "ERROR: AddressSanitizer" not in out and "runtime error" not in out, out[-4000:]
