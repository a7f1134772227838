"""Build libtwg.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache)."""
from __future__ import annotations

import os
import subprocess
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(_HERE)
SOURCES = ["api.cu", "api_track.cu", "api_sim.cu", "api_extra.cu", "host_core.cu", "k_relax.cu", "k_stamp.cu",
           "k_path.cu", "k_track.cu", "k_sim.cu", "nccl_link.cu", "api_shard.cu"]
HEADERS = ["twg_internal.cuh", "twg_kernels.cuh", "api_host.cuh"]
OUT = os.path.join(_HERE, "libtwg.so")

# -fmad=false: no FMA contraction anywhere (bit-exact parity with the oracle);
# default IEEE division/sqrt and no flush-to-zero (no --use_fast_math).
NVCC_FLAGS = ["-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-fmad=false",
              "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared"]


LINK_LIBS = ["-ldl"]


def _nvcc():
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if p and (os.path.sep not in p or os.path.exists(p)):
            return p
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(_HERE, "csrc", s) for s in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "twg.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile every translation unit in parallel (one nvcc per file), then link libtwg.so (or `out`, with
    extra -D `defines`: variant builds for timing experiments)."""
    OUT = out or globals()["OUT"]
    if out is None and not force and not needs_build():
        return OUT
    from concurrent.futures import ThreadPoolExecutor
    import tempfile
    inc = ["-I", os.path.join(ROOT, "include")]
    comp = [f for f in NVCC_FLAGS if f != "-shared"] + [f"-D{d}" for d in defines]
    with tempfile.TemporaryDirectory(prefix="twg_build_") as tmp:
        objs = [os.path.join(tmp, os.path.splitext(s)[0] + ".o") for s in SOURCES]

        def one(k):
            cmd = [_nvcc()] + comp + inc + ["-c", os.path.join(_HERE, "csrc", SOURCES[k]), "-o", objs[k]]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed on {SOURCES[k]}:\n{r.stdout}{r.stderr}")
            if r.stderr.strip() and verbose:
                print(r.stderr, file=sys.stderr)

        with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
            list(ex.map(one, range(len(SOURCES))))
        cmd = [_nvcc()] + NVCC_FLAGS + objs + LINK_LIBS + ["-o", OUT + ".tmp"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
