"""Build the CPU oracle shared library (plain C, gcc).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.
"""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "fskmc_oracle.c")
LIB = os.path.join(HERE, "_fskmc_oracle.so")


def build(force: bool = False) -> str:
    if os.environ.get("ORC_LIB"):          # an alternative build (tools/oracle_timing.py: OpenMP)
        return os.environ["ORC_LIB"]
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    # -ffp-contract=off: the clock arithmetic is the IEEE operation sequence of
    # DESIGN.md §3 (no fused multiply-add contraction).
    cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           "-Wall", "-Wno-unused-function", "-o", LIB + ".tmp", SRC, "-lm"]
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_openmp(path: str) -> str:
    """The same source with -fopenmp (the cells of a colour on all host cores; timing only)."""
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                           "-fopenmp", "-Wall", "-Wno-unused-function", "-o", path, SRC, "-lm"])
    return path


if __name__ == "__main__":
    print(build(force=True))
