"""Per-kernel timing of the device feature front-end at 640x480 (run under
`ncu --metrics gpu__time_duration.sum` for the launch list, or plain for the
wall-clock of detect / match / store calls)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import pyoracle as O  # noqa: E402  (synthetic frames only)
from paper_1603_08161_b200.abi import FeatureParams, Frame, Intrinsics  # noqa: E402
from paper_1603_08161_b200.wfk import Context  # noqa: E402

K = Intrinsics.make(560, 560, 319.5, 239.5, 640, 480)
ctx = Context(0)
d, c = O.synth_render(K, amplitude=0.5)
fr = Frame(K, d, c)
ctx.upload_frame(fr)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for _ in range(3):
    feats, nk = ctx.detect_features()
t0 = time.perf_counter()
for _ in range(reps):
    feats, nk = ctx.detect_features()
t1 = time.perf_counter()
print(f"detect: {len(feats)} features / {nk} keypoints, {(t1 - t0) / reps * 1e3:.3f} ms per call (host clock)")
st = np.concatenate([feats] * 10)
st["frame_id"] = np.repeat(np.arange(10), len(feats))
pred = np.tile(np.array([0.0, 0.0, 1.2]), (len(st), 1))
for _ in range(3):
    ctx.match_features(feats, st, pred, K)
t0 = time.perf_counter()
for _ in range(reps):
    m = ctx.match_features(feats, st, pred, K)
t1 = time.perf_counter()
print(f"match: {len(m)} matches vs a {len(st)}-entry store, {(t1 - t0) / reps * 1e3:.3f} ms per call (host clock)")
ctx.close()
