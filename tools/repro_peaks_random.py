import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2212_09460_b200 import ld
rng = np.random.default_rng(9)
NT = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for trial in range(NT):
    b = int(rng.integers(1, 4))
    n_t, n_r = int(rng.integers(1, 40)), int(rng.integers(1, 700))
    acc = rng.integers(0, int(rng.integers(1, 8)), size=(b, n_t, n_r)).astype(np.uint32)
    ht, hr = int(rng.integers(0, 5)), int(rng.integers(0, 30))
    mv, k = int(rng.integers(0, 5)), int(rng.choice([1, 2, 4, 7, 64, 1024]))
    print(trial, b, n_t, n_r, ht, hr, mv, k, flush=True)
    peaks, npk = ld.hough_peaks(torch.from_numpy(acc.view(np.int32)).cuda(), ht, hr, mv, k)
    torch.cuda.synchronize()
    L = ld.lib()
    if hasattr(L, "ld_debug_error_line"):
        L.ld_debug_error_line.restype = ctypes.c_int
        print("  debug line", L.ld_debug_error_line(), flush=True)
print("ok")
