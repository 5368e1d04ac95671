"""Source-level guard for programmatic dependent launch: a kernel launched with the
programmatic-serialization attribute may start before its predecessor has finished, so it MUST
call pdl_wait() before it touches anything -- every kernel that can reach launch_pdl() is checked
to contain the wait (a missing one is a race that the GPU tests need not hit)."""
import os
import re

CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                    "paper_1105_4002_b200", "csrc")


def _kernel_bodies(src):
    """name -> text from the kernel's __global__ to the next __global__ (or end of file)."""
    out = {}
    parts = re.split(r"(?=__global__)", src)
    for p in parts[1:]:
        m = re.search(r"\b(\w+_kernel)\s*\(", p)
        if m:
            out.setdefault(m.group(1), p)
    return out


def _function_body(src, name):
    i = src.index(name)
    j = src.index("{", i)
    depth, k = 0, j
    while True:
        depth += src[k] == "{"
        depth -= src[k] == "}"
        k += 1
        if depth == 0:
            return src[j:k]


def test_every_pdl_launched_kernel_waits():
    spmv = open(os.path.join(CSRC, "spmv.cu")).read()
    tv = open(os.path.join(CSRC, "tv.cu")).read()
    launched = set()
    # spmv.cu: launch_pdl is called from launch_spmv16s with the kernels of the dispatch tables
    assert spmv.count("launch_pdl(") == 2
    for fn in ("static cudaError_t dispatch16s(", "static cudaError_t dispatch16s_lo("):
        launched |= set(re.findall(r"\b(\w+_kernel)\b", _function_body(spmv, fn)))
    # tv.cu: launch_pdl(k, ...) with k = tv_row_kernel<...>, and launch_pdl(tv_kernel<...>, ...)
    for m in re.finditer(r"launch_pdl\(\s*(\w+)", tv):
        name = m.group(1)
        if name == "k":  # the nearest "auto k = <kernel><...>" above the launch
            name = re.findall(r"auto k = (\w+_kernel)<", tv[:m.start()])[-1]
        launched.add(name)
    assert {"spmv16s_kernel", "spmv16z_kernel", "tv_row_kernel", "tv_kernel"} <= launched, launched
    bodies = {}
    bodies.update(_kernel_bodies(spmv))
    bodies.update(_kernel_bodies(tv))
    for name in sorted(launched):
        assert name in bodies, name
        assert "pdl_wait()" in bodies[name], f"{name} is launched with launch_pdl but never waits"
    # and no other file launches with the attribute
    for f in os.listdir(CSRC):
        if f.endswith(".cu") and f not in ("spmv.cu", "tv.cu"):
            assert "launch_pdl(" not in open(os.path.join(CSRC, f)).read(), f
