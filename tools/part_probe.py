import sys, time, os
sys.argv = ["bench.py", "--partitioned"] + sys.argv[1:]
sys.path.insert(0, ".")
import bench
# monkeypatch to time each solve by wall clock
from paper_1603_08161_b200 import wfk
orig = wfk.Context.solve_coarse_to_fine_dist
def timed(self, pose, p):
    import ctypes
    t0 = time.perf_counter()
    r = orig(self, pose, p)
    print(f"[probe] dist solve wall {1e3*(time.perf_counter()-t0):.1f} ms, trace {len(r)} entries", file=sys.stderr)
    return r
wfk.Context.solve_coarse_to_fine_dist = timed
bench.main()
