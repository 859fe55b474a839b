"""Measurement: path counters of the integer-max scaled recursion (FASE_ITERATE_STATS build)."""
import ctypes, runpy, sys
sys.argv = ["bench.py", "--steps", "1", "--warmup", "1", "--no-cpu-baseline"] + sys.argv[1:]
try:
    runpy.run_path("bench.py", run_name="__main__")
except SystemExit:
    pass
from paper_2204_14194_b200 import _native
lib = ctypes.CDLL(str(_native.library_path()))
out = (ctypes.c_ulonglong * 8)()
lib.fase_iterate_stats(out)
names = ["block_iterations", "warp_exact_scans", "tie_pass_exact", "mispredicted", "warp_iterations", "tie_pass_spread", "-", "-"]
print("STATS", dict(zip(names, list(out))))
