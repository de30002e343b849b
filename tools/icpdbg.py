import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from test_gpu_icp import *
from paper_1603_08161_b200.wfk import Context
ctx = Context(0)
vol = fused_volume()
d1, c1 = O.synth_render(K)
fr = Frame(K, d1, c1)
for it in (1, 2, 3):
    ref, got = run_both(ctx, vol, fr, Pose.make(), IcpParams.make(max_iters=it))
    print(it, "ref", ref.degraded, ref.iterations, ref.rms, ref.pose.vector(), "got", got.degraded, got.iterations, got.rms, got.pose.vector())
b = ctx.rasterize(K, download=True)
print("valid px", np.isfinite(b.depth).sum() if hasattr(b,'depth') else b)
m = ctx.backproject_depth(download=True)
print(type(m), [k for k in dir(m) if not k.startswith('_')][:10])
