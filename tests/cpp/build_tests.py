"""Builds tests/cpp/test_api (the C++ host API checked against the CPU
oracle) with g++ against the in-tree libdfm_b200.so and oracle/_build/
libdfm_oracle.so.  The rpath is relative to the binary, so the build travels
with the repository snapshot to a GPU box.  Called by __graft_entry__.build()."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "test_api.cpp")
    out = os.path.join(HERE, "test_api")
    deps = [src, os.path.join(ROOT, "include", "fastmnmf_b200.hpp"), os.path.join(ROOT, "include", "dfm_b200.h"),
            os.path.join(ROOT, "oracle", "dfm_oracle.h")]
    libs = [os.path.join(ROOT, "paper_2605_19388_b200", "libdfm_b200.so"),
            os.path.join(ROOT, "oracle", "_build", "libdfm_oracle.so")]
    if not force and os.path.exists(out) and all(os.path.getmtime(out) >= os.path.getmtime(d) for d in deps + libs):
        return out
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(ROOT, "oracle"), src, "-o", out,
           "-L", os.path.join(ROOT, "paper_2605_19388_b200"), "-ldfm_b200",
           "-L", os.path.join(ROOT, "oracle", "_build"), "-ldfm_oracle",
           "-Wl,-rpath,$ORIGIN/../../paper_2605_19388_b200:$ORIGIN/../../oracle/_build"]
    subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    print(build(force=True))
