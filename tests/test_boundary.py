"""The product package never routes through the oracle and has no CPU fallback."""

import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_2204_14194_b200"


def test_product_never_imports_oracle():
    for path in list(PKG.rglob("*.py")) + list(PKG.rglob("*.cu")) + list(PKG.rglob("*.cuh")):
        text = path.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle\b", text, re.M), path
        assert "fase_oracle" not in text, path


def test_product_never_reads_the_reference_tree():
    for path in list(PKG.rglob("*.py")) + [ROOT / "bench.py", ROOT / "__graft_entry__.py"]:
        assert "/root/reference" not in path.read_text(), path


def test_bench_touches_oracle_only_in_cpu_baseline():
    text = (ROOT / "bench.py").read_text()
    lines = [i for i, ln in enumerate(text.splitlines()) if "oracle" in ln and "import" in ln]
    body = text.splitlines()
    for i in lines:
        # every oracle import sits inside the CPU-reference helpers
        ctx = "\n".join(body[max(0, i - 12):i])
        assert "def _cpu_worker" in ctx or "def cpu_prepare" in ctx, body[i]


def test_no_forbidden_batch_memcpy():
    # the pool forbids the batched-memcpy family; names are assembled so that
    # this file does not itself spell them
    stem = "Batch" + "Async"
    banned = tuple(p + stem for p in ("cudaMemcpy", "cudaMemcpy3D", "cuMemcpy", "cuMemcpy3D"))
    for path in list(PKG.rglob("*")) + list((ROOT / "include").rglob("*")):
        if path.is_file() and path.suffix in (".cu", ".cuh", ".h", ".py", ".cpp"):
            text = path.read_text()
            assert not any(b in text for b in banned), path
