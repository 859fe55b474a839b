"""Register / spill budget of the hot recursion shapes (CPU: nvcc cross-compile).

The benchmarked recursions run at their register ceilings (config 1: 256
threads x 18 elements at four CTAs per SM = 64 registers; config 4: 256 x 32 at
two = 128; configs 2 / 3: the chunked 256 x 18 / 128 x 16 at 80). One more live
value there spills in the update loop: the block index loaded from a dispatch
order once cost config 1 a 13% slowdown (16 -> 120 spill bytes). This
test compiles csrc/iterate.cu with ptxas -v and holds each shape to its budget.
"""

import re
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CSRC = ROOT / "paper_2204_14194_b200" / "csrc"

# (template arguments as c++filt prints them) -> (registers, max spill-store bytes)
BUDGET = {
    # config 1, scaled: 256 x 18, four CTAs per SM
    "<256, 18, 4, false, false, false, 1, true, 0, 0>": (64, 32),
    # config 4, scaled: 256 x 32, two CTAs per SM
    "<256, 32, 2, false, false, false, 1, true, 0, 0>": (128, 8),
    # config 2, chunked exact: 256 x 18, three CTAs per SM
    "<256, 18, 3, true, true, false, 1, false, 0, 0>": (80, 48),
    # config 3, chunked exact: 128 x 16, six CTAs per SM
    "<128, 16, 6, true, true, false, 1, false, 0, 0>": (80, 8),
}


@pytest.fixture(scope="module")
def ptxas_report(tmp_path_factory):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(nvcc).exists():
        pytest.skip("nvcc not available")
    out = tmp_path_factory.mktemp("ptxas") / "iterate.o"
    proc = subprocess.run(
        [nvcc, "-gencode=arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
         "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", f"-I{CSRC}", "-Xptxas", "-v", "-c",
         str(CSRC / "iterate.cu"), "-o", str(out)],
        capture_output=True, text=True)
    assert proc.returncode == 0, proc.stderr[-2000:]
    res, cur = {}, None
    for line in proc.stderr.splitlines():
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
            res[cur] = {"spill": 0, "reg": None}
            continue
        m = re.search(r"(\d+) bytes spill stores", line)
        if m and cur:
            res[cur]["spill"] = int(m.group(1))
        m = re.search(r"Used (\d+) registers", line)
        if m and cur:
            res[cur]["reg"] = int(m.group(1))
    names = subprocess.run(["c++filt"], input="\n".join(res), capture_output=True,
                           text=True).stdout.splitlines()
    out = {}
    for mangled, plain in zip(res, names):
        if "fase_iterate_kernel<" in plain:
            out[plain.split("fase_iterate_kernel")[1].split("(")[0]] = res[mangled]
    return out


@pytest.mark.parametrize("shape", sorted(BUDGET))
def test_hot_recursion_shapes_within_register_budget(ptxas_report, shape):
    regs, spill = BUDGET[shape]
    got = ptxas_report.get(shape)
    assert got is not None, f"{shape} not instantiated"
    assert got["reg"] <= regs, (shape, got)
    assert got["spill"] <= spill, (shape, got)
