"""Build libtsim.so in-tree for sm_100a (nvcc, no JIT cache)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRCS = ["csrc/tsim_kernels.cu", "csrc/tsim_rows.cu", "csrc/tsim_api.cu", "csrc/tsim_readers.cu", "csrc/tsim_partition.cpp",
        "csrc/tsim_text.cpp"]
SO = os.path.join(HERE, "libtsim.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "-ldl"]


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(HERE, s) for s in SRCS] + [
        os.path.join(HERE, "csrc", "tsim_internal.h"),
        os.path.join(HERE, "csrc", "tsim_host.h"),
        os.path.join(HERE, "csrc", "tsim_device.cuh"),
        os.path.join(os.path.dirname(HERE), "include", "tsim.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return SO
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc] + NVCC_FLAGS + [os.path.join(HERE, s) for s in SRCS] + ["-o", SO]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    if verbose:
        print(r.stderr)
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
        # register / spill / shared-memory report per kernel (compile times
        # dropped so the file changes only with the code)
        f.write("".join(ln for ln in r.stderr.splitlines(True) if "Compile time" not in ln))
    return SO


CHECKED_SO = os.path.join(os.path.dirname(HERE), "build", "checked", "libtsim.so")


def build_checked(force: bool = False) -> str:
    """The same sources with -DTS_CHECKED (invariant counters in the row
    kernel, ts_debug_checks): a debug library for tests, never benchmarked."""
    deps = [os.path.join(HERE, s) for s in SRCS] + [SO]
    if (not force and os.path.exists(CHECKED_SO) and
            all(os.path.getmtime(d) <= os.path.getmtime(CHECKED_SO) for d in deps if os.path.exists(d))):
        return CHECKED_SO
    os.makedirs(os.path.dirname(CHECKED_SO), exist_ok=True)
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc] + NVCC_FLAGS + ["-DTS_CHECKED"] + \
        [os.path.join(HERE, s) for s in SRCS] + ["-o", CHECKED_SO]
    cmd = [c for i, c in enumerate(cmd) if not (c == "-Xptxas" and cmd[i + 1:i + 2] == ["-v"])
           and not (c == "-v" and cmd[i - 1] == "-Xptxas")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc (checked) failed:\n" + r.stdout + r.stderr)
    return CHECKED_SO


if __name__ == "__main__":
    print(build(force=True, verbose=True))
