"""e2e probe (GPU box): device-resident inference vs the synchronous host call
vs the pipelined submit/wait, per-step ms, on one config."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2004_10908_b200 as sd  # noqa: E402
import sdnngen as g  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
n, L, B = bench.CONFIGS[cfg]
net = sd.Net.from_spec(g.rn_spec(n, L), fmt="ell", threads=8, device=0)
rp, idx = g.ms_inputs(n, B)
rp_h = torch.from_numpy(rp).pin_memory().numpy()
idx_h = torch.from_numpy(idx).pin_memory().numpy()
rp_t, idx_t = torch.from_numpy(rp).cuda(), torch.from_numpy(idx).cuda()
for _ in range(2):
    net.infer_torch(rp_t, idx_t)
torch.cuda.synchronize()
K = 5
t = time.perf_counter()
for _ in range(K):
    net.infer_torch(rp_t, idx_t)
torch.cuda.synchronize()
dev = (time.perf_counter() - t) / K
net.infer(rp_h, idx_h, None)
t = time.perf_counter()
for _ in range(3):
    net.infer(rp_h, idx_h, None)
syn = (time.perf_counter() - t) / 3
for K in (2, 4, 8):
    net.infer_wait(net.infer_submit(rp_h, idx_h))
    t = time.perf_counter()
    tk = [net.infer_submit(rp_h, idx_h)]
    sub = [time.perf_counter() - t]
    for k in range(K):
        if k + 1 < K:
            t0 = time.perf_counter()
            tk.append(net.infer_submit(rp_h, idx_h))
            sub.append(time.perf_counter() - t0)
        net.infer_wait(tk[k])
    pipe = (time.perf_counter() - t) / K
    print(f"{cfg}: device {dev*1e3:.1f} ms  sync {syn*1e3:.1f} ms  pipelined(K={K}) {pipe*1e3:.1f} ms  "
          f"submit call {1e3*np.mean(sub):.1f} ms", flush=True)
t = time.perf_counter()
from paper_2004_10908_b200 import lib  # noqa: E402
print("nnz", idx.size, "bytes", idx.nbytes + rp.nbytes)
# (a) device loop with a concurrent 2 GB host->device copy per step on a side stream
side = torch.cuda.Stream()
dst = torch.empty(idx.size, dtype=torch.int32, device="cuda")
src = torch.from_numpy(idx_h)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    with torch.cuda.stream(side):
        dst.copy_(src, non_blocking=True)
    net.infer_torch(rp_t, idx_t)
torch.cuda.synchronize()
print(f"device + concurrent 2 GB H2D: {(time.perf_counter() - t) / 3 * 1e3:.1f} ms", flush=True)
# (b) synchronous host call without host validation
net2 = sd.Net.from_spec(g.rn_spec(n, L), fmt="ell", threads=8, device=0, flags=sd.SDNN_F_TRUST_INPUT)
net2.infer(rp_h, idx_h, None)
t = time.perf_counter()
for _ in range(3):
    net2.infer(rp_h, idx_h, None)
print(f"sync, SDNN_F_TRUST_INPUT: {(time.perf_counter() - t) / 3 * 1e3:.1f} ms", flush=True)
