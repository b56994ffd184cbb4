"""Cluster-voting repro: one frame of random edges voted with and without the
thread-block cluster path, checked against each other; each case in its own
process (a device fault is sticky).  python tools/repro_cluster.py"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CASE = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2212_09460_b200 import ld, synth
n_theta, b, want_hint = %d, %d, %d
c, s = synth.q15_table(n_theta)
rng = np.random.default_rng(1)
w, h = 301, 203
n = 4099
el = np.zeros((b, 4100), np.uint32)
for i in range(b):
    xs, ys = rng.integers(0, w, n), rng.integers(0, h, n)
    el[i, :n] = (ys.astype(np.uint32) << 16) | xs.astype(np.uint32)
e = torch.from_numpy(el.view(np.int32)).cuda()
cnt = torch.full((b,), n, dtype=torch.int32, device="cuda")
a0 = ld.hough_accumulate(e, cnt, 4100, w, h, c, s, flags=ld.LD_VOTE_NO_CLUSTER)
torch.cuda.synchronize()
r = ld.hough_accumulate(e, cnt, 4100, w, h, c, s, want_hint=bool(want_hint))
a1 = r[0] if want_hint else r
torch.cuda.synchronize()
print("OK" if torch.equal(a0, a1) else "MISMATCH")
'''
for nt in ((1,) if os.environ.get("QUICK") else (1, 2, 180)):
    for b in ((1,) if os.environ.get("QUICK") else (1, 4)):
        for hint in ((0,) if os.environ.get("QUICK") else (0, 1)):
            r = subprocess.run([sys.executable, "-c", CASE % (nt, b, hint)], capture_output=True,
                               text=True, env=dict(os.environ, CUDA_LAUNCH_BLOCKING="1"))
            out = (r.stdout.strip().splitlines() or [""])[-1]
            err = [ln for ln in r.stderr.splitlines() if "Error" in ln or "error" in ln][-1:]
            print("n_theta=%d batch=%d hint=%d -> %s %s" % (nt, b, hint, out, err))
