"""Register-spill guard for the hot kernels (build-level regression test, no GPU): the stencil and
SpMV instantiations the passes launch must compile for sm_100a without spills (a spilling stencil
ran 29 -> 37 us at c2 once, from a launch-bounds slip)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1105_4002_b200", "csrc")

# (mangled-name pattern, spill bytes allowed)
HOT = {
    "tv.cu": [
        (r"tv_kernelINS_8SrcPlainELi0ELi5EiE", 0),       # tvr_objective_grad: W1 | G
        (r"tv_kernelINS_8SrcPlainELi0ELi69EiE", 0),      # solver gradient + stop test
        (r"tv_kernelINS_8SrcPlainELi0ELi65EiE", 0),      # UPN stop test at x_{k+1}
        (r"tv_kernelINS_12SrcMomentumXILb1EEELi0ELi15EiE", 0),  # UPN momentum point (hi + lo state)
        (r"tv_kernelINS_12SrcMomentumXILb1EEELi0ELi143EiE", 0),  # same, device-side control
        (r"tv_kernelINS_8SrcTrialELi1ELi0EiE", 0),       # trial points
        (r"tv_kernelINS_8SrcTrialELi1ELi32EiE", 0),
        (r"tv_kernelINS_8SrcTrialELi1ELi64EiE", 0),
        (r"tv_kernelINS_9SrcTrialXILb1EEELi1ELi0EiE", 0),  # BT trials (hi + lo state)
        (r"tv_kernelINS_9SrcTrialXILb1EEELi1ELi32EiE", 0),
        # row-tiled stencil (K = 4; one-warp rows: c2, two-warp rows: c3 / c5)
        (r"tv_row_kernelINS_8SrcPlainELi0ELi5ELi4ELi7ELi1E", 0),   # tvr_objective_grad
        (r"tv_row_kernelINS_8SrcPlainELi0ELi5ELi4ELi7ELi2E", 0),
        (r"tv_row_kernelINS_8SrcPlainELi0ELi69ELi4ELi7ELi1E", 0),  # solver gradient + stop test
        (r"tv_row_kernelINS_8SrcPlainELi0ELi69ELi4ELi7ELi2E", 0),
        (r"tv_row_kernelINS_8SrcTrialELi1ELi0ELi4ELi7ELi1E", 0),   # trial points
        (r"tv_row_kernelINS_8SrcTrialELi1ELi64ELi4ELi7ELi2E", 0),
        (r"tv_row_kernelINS_12SrcMomentumXILb1EEELi0ELi15ELi4ELi7ELi1E", 0),  # UPN momentum point
        (r"tv_row_kernelINS_9SrcTrialXILb1EEELi1ELi32ELi4ELi7ELi1E", 0),     # UPN BT trial
    ],
    "spmv.cu": [
        (r"spmv16s_kernelILi2ELb1ELi512ELb0ELb1ELi0E", 0),   # sliced ELL: c2 A and A^T passes
        (r"spmv16s_kernelILi2ELb1ELi1024ELb0ELb1ELi0E", 0),  # c3 A^T pass (wide CTA)
        (r"spmv16s_kernelILi2ELb1ELi1024ELb1ELb1ELi0E", 0),  # c3 A pass (partly staged window)
        (r"spmv16p_kernelILi8ELi3ELb1E", 0),   # padded per-row kernel (TVR_SPMV_SELL=0)
        (r"spmv32s_kernelILi2ELi512ELi0ELb0EE", 0),  # int32 sliced ELL: c5 A pass
        (r"spmv32s_kernelILi3ELi512ELi0ELb0EE", 8),  # int32 sliced ELL: c5 / f2 A^T pass
        (r"spmv32s_kernelILi3ELi1024ELi0ELb0EE", 0),  # c5 A / A^T (1024-thread CTAs)
        (r"spmv16s_kernelILi2ELb1ELi1024ELb0ELb1ELi1EE", 0),  # extended-precision UPN A pass (c3 parts)
        (r"spmv16s_kernelILi2ELb1ELi1024ELb0ELb1ELi2EE", 16),  # same, lo window staged (c2; 8 B)
        (r"spmv16z_kernelILi2ELi1ELi1024EE", 0),  # slice-shared operator, 2 slices per pass
        (r"spmv16p_kernelILi4ELi3ELb1E", 0),   # c2 A^T pass
        (r"spmv16p_kernelILi8ELi2ELb0E", 0),   # c3 A pass (global gather)
        (r"spmv32p_kernelILi4ELi2E", 0),       # non-separable
        (r"spmv32p_kernelILi8ELi2E", 0),
    ],
}


def _spills(src):
    out = subprocess.run(
        ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xptxas", "-v",
         "-c", os.path.join(CSRC, src), "-o", os.devnull],
        capture_output=True, text=True, check=True).stderr
    res, cur = {}, None
    for line in out.splitlines():
        m = re.search(r"Compiling entry function '([^']+)'", line)
        if m:
            cur = m.group(1)
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            res[cur] = int(m.group(1)) + int(m.group(2))
    return res


@pytest.mark.parametrize("src", sorted(HOT))
def test_hot_kernels_do_not_spill(src):
    sp = _spills(src)
    for pat, allowed in HOT[src]:
        hits = [k for k in sp if re.search(pat, k)]
        assert hits, f"{pat} not compiled"
        for k in hits:
            assert sp[k] <= allowed, f"{k} spills {sp[k]} bytes"
