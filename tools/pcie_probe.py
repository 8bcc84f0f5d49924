"""PCIe copy ceilings for the e2e leg (diagnostics): 51 MB H2D alone, 52 MB
D2H alone, and both at once on two streams, pinned host memory."""
import json
import time

import torch

N_IN, N_OUT, K = 51_216_384, 52_055_820, 20
h_in = torch.empty(N_IN, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N_OUT, dtype=torch.uint8).pin_memory()
d_in = torch.empty(N_IN, dtype=torch.uint8, device="cuda")
d_out = torch.empty(N_OUT, dtype=torch.uint8, device="cuda")
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(K):
        if h2d:
            with torch.cuda.stream(s_in):
                d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s_out):
                h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / K * 1e3


for _ in range(2):
    run(True, True)
res = {"h2d_ms": run(True, False), "d2h_ms": run(False, True), "both_ms": run(True, True)}
res["h2d_GBps"] = N_IN / res["h2d_ms"] / 1e6
res["d2h_GBps"] = N_OUT / res["d2h_ms"] / 1e6
print(json.dumps(res))
