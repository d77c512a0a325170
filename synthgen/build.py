"""Build synthgen/libsynthgen.so (device twin of synthgen/host.py) for sm_100a."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build(verbose: bool = False) -> str:
    src = os.path.join(HERE, "csrc", "synthgen.cu")
    out = os.path.join(HERE, "libsynthgen.so")
    if os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(src):
        return out
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-shared", "-Xcompiler",
           "-fPIC,-fvisibility=hidden", "-o", out + ".tmp", src]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(True))
