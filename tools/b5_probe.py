"""Run the libld.so B5 shared-atomic microbenchmark once per mode (for an ncu
capture of smem_atomic_bench_kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2212_09460_b200 import ld  # noqa: E402

scratch = torch.empty((ld.ld_device_sm_count() * 2 * 32,), dtype=torch.int32, device="cuda")
for mode in (0, 1, 2):
    ld.ld_bench_smem_atomics(mode, 4096 if mode < 2 else 256, 1, scratch)
torch.cuda.synchronize()
print("ok")
