"""Time one K = 1 layer as the model runs it (dec4.r0.proj: level 0 of the
bench's 8-scan pack, 96 + 32 concatenated channels -> 96, BN):
SCB_DENSE_K1=1 (scb_conv_pointwise) or 0 (gather-form identity map)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10319_b200 as sc  # noqa: E402
from paper_2204_10319_b200 import execution as X  # noqa: E402

n = int(os.environ.get("N", 1000366))
ca, cb, co = (int(os.environ.get(k, d)) for k, d in (("CA", 96), ("CB", 32), ("COUT", 96)))
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.standard_normal((n, ca)).astype(np.float16)).cuda()
skip = torch.from_numpy(rng.standard_normal((n, cb)).astype(np.float16)).cuda() if cb else None
w = sc.WeightTensor(rng.normal(0, 0.05, (1, ca + cb, co)).astype(np.float32), 1, 3)
ep = {"scale": torch.rand(co, device="cuda") + 0.5, "shift": torch.rand(co, device="cuda") - 0.5}
opts = sc.ExecOptions(dataflow="fused")
for _ in range(5):
    X._run_fused(x, None, w, opts, ep, skip)
torch.cuda.synchronize()
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    X._run_fused(x, None, w, opts, ep, skip)
e.record()
torch.cuda.synchronize()
print(f"pointwise {ca}+{cb}->{co} ({n} rows): {a.elapsed_time(e) / 20:.4f} ms  "
      f"dense={os.environ.get('SCB_DENSE_K1', '1')}")
