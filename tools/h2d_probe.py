"""Host->device copy bandwidth from pinned memory: one stream vs several
concurrent streams (copy engines), chunk sizes of the e2e path."""
import time
import torch

N = 236 * 1024 * 1024
host = torch.empty(N, dtype=torch.uint8).pin_memory()
dev = torch.empty(N, dtype=torch.uint8, device="cuda")
for streams in (1, 2, 4):
    for chunk_mb in (8, 29.5, 64):
        chunk = int(chunk_mb * 1024 * 1024)
        ss = [torch.cuda.Stream() for _ in range(streams)]
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            i = 0
            for off in range(0, N, chunk):
                with torch.cuda.stream(ss[i % streams]):
                    dev[off:off + chunk].copy_(host[off:off + chunk], non_blocking=True)
                i += 1
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        print({"streams": streams, "chunk_mb": chunk_mb, "GB/s": round(N / dt / 1e9, 1)})
d2h = torch.empty(N, dtype=torch.uint8).pin_memory()
torch.cuda.synchronize()
t0 = time.perf_counter()
d2h.copy_(dev, non_blocking=True)
torch.cuda.synchronize()
print({"d2h_GB/s": round(N / (time.perf_counter() - t0) / 1e9, 1)})
