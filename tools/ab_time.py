"""A/B timing of the three stages on one workload with the libld.so named by
the LD_LIB environment variable (default: the in-tree build).  Prints one JSON
line: mean ms per stage over --reps serialised steps (CUDA events).

    LD_LIB=build/libld_variant.so python tools/ab_time.py --workload cfg3
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2212_09460_b200 import ld, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg3")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
cfg = synth.CONFIGS[a.workload]
B, W, H = cfg.batch, cfg.width, cfg.height
c, s = synth.q15_table(cfg.n_theta)
frames = synth.gen_batch(a.workload, 0, B) if B > 1 else synth.gen_frame(a.workload, 0)[None]
pitch = ld._round_up(W, 16)
g = torch.zeros((B, H, pitch), dtype=torch.uint8, device="cuda")
g[:, :, :W] = torch.from_numpy(frames).cuda()
img = ld.make_image(W, H, pitch, H * pitch, B)
stride = ld._round_up(H * (W - 2), 4)
n_rho = 2 * ld.ld_rho_offset(W, H) + 1
edges = torch.empty((B, stride), dtype=torch.int32, device="cuda")
cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
acc = torch.empty((B, cfg.n_theta, n_rho), dtype=torch.int32, device="cuda")
hb = ld.ld_hough_hint_bytes(B, W, H, cfg.n_theta)
hint = torch.empty((hb,), dtype=torch.uint8, device="cuda")
wb = ld.ld_hough_peaks_workspace_bytes(B, cfg.n_theta, n_rho, cfg.k)
ws = torch.empty((wb,), dtype=torch.uint8, device="cuda")
pk = torch.empty((B, cfg.k, 3), dtype=torch.int32, device="cuda")
npk = torch.empty((B,), dtype=torch.int32, device="cuda")
ts = []
for i in range(a.reps + 3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    ld.ld_sobel_binarize(g, img, cfg.threshold, None, edges, stride, cnt)
    ev[1].record()
    ld.ld_hough_accumulate_hint(edges, cnt, stride, B, W, H, cfg.n_theta, c, s, acc, hint, hb)
    ev[2].record()
    ld.ld_hough_peaks_hinted(acc, B, cfg.n_theta, n_rho, cfg.half_theta, cfg.half_rho,
                             cfg.min_votes, cfg.k, hint, hb, pk, npk, ws, wb)
    ev[3].record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append([ev[j].elapsed_time(ev[j + 1]) for j in range(3)])
t = np.array(ts).mean(axis=0)
print(json.dumps({"lib": os.environ.get("LD_LIB", "in-tree"), "workload": a.workload,
                  "sobel_ms": t[0], "vote_ms": t[1], "peaks_ms": t[2],
                  "peaks_sum": int(pk.sum().item())}))
