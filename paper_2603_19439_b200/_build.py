"""In-tree build of the CUDA library (sm_100a) behind include/spectrack_gpu.h."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libspectrack_b200.so")
# host library: stream generators + the update-batch wire format (include/spectrack_stream.h)
STREAM_LIB = os.path.join(HERE, "libspectrack_stream.so")
STREAM_SOURCES = ["csrc/streamgen.cpp", "../include/spectrack_stream.h"]
SOURCES = ["csrc/session.cu"]
HEADERS = ["csrc/common.cuh", "csrc/dmma.cuh", "csrc/spmm.cuh", "csrc/smalllin.cuh", "csrc/rng.cuh",
           "csrc/ingest.cuh", "csrc/stepk.cuh", "csrc/eigsolve.cuh", "csrc/shard.cuh", "csrc/lanczos.cuh", "csrc/nccl_comm.cuh", "csrc/trackers.cuh", "csrc/metrics.cuh", "../include/spectrack_gpu.h"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(os.path.join(HERE, f)) > t for f in SOURCES + HEADERS)


def _stream_stale() -> bool:
    if not os.path.exists(STREAM_LIB):
        return True
    t = os.path.getmtime(STREAM_LIB)
    return any(os.path.getmtime(os.path.join(HERE, f)) > t for f in STREAM_SOURCES)


def build_stream(force: bool = False) -> str:
    if force or _stream_stale():
        cmd = ["g++", "-std=c++17", "-O3", "-fopenmp", "-fPIC", "-shared", "-Wall", "-Wextra",
               "-o", STREAM_LIB, os.path.join(HERE, "csrc/streamgen.cpp")]
        subprocess.run(cmd, check=True)
    return STREAM_LIB


def build(force: bool = False) -> str:
    build_stream(force)
    if force or _stale():
        nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
        cmd = [nvcc, *NVCC_FLAGS, "-o", LIB, *[os.path.join(HERE, s) for s in SOURCES], "-lcusolver", "-ldl"]
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
