"""Time one transposed k2 layer (level 1 -> level 0 of the bench's 8-scan
pack, 96 -> 96 channels) as the model runs it: one-hot tile order or not."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10319_b200 as sc  # noqa: E402
from paper_2204_10319_b200.mapping import reorder_by_presence  # noqa: E402
from bench import load_scans, pack  # noqa: E402

c, f, b = pack(load_scans(range(8)))
rng = np.random.default_rng(0)
t0 = sc.SparseTensor(torch.from_numpy(c.astype(np.int32)).cuda(), np.zeros((c.shape[0], 1), np.float32), 1, b, 8)
p = reorder_by_presence(t0.coordset, 3, "hash")
n = p.num_points
x = sc.SparseTensor._wrap(torch.from_numpy(rng.standard_normal((n, 96)).astype(np.float16)).cuda(), 1, b, 8, p)
wd = sc.WeightTensor(rng.normal(0, 0.05, (8, 96, 96)).astype(np.float32), 2, 3)
wu = sc.WeightTensor(rng.normal(0, 0.05, (8, 96, 96)).astype(np.float32), 2, 3)
cache = {}
opts = sc.ExecOptions(dataflow="fused", index_kind="hash")
if os.environ.get("L1_REORDER", "0") == "1":   # the model's level 1: presence-relabelled
    from paper_2204_10319_b200.execution import prepare_reordered_level
    prepare_reordered_level(p, sc.LayerSpec(2, 2, 96, 96), opts)
d = sc.sparse_conv_forward(x, wd, sc.LayerSpec(2, 2, 96, 96, reuse_key="d"), None, cache, opts)
spec = sc.LayerSpec(2, 1, 96, 96, transposed=True, reuse_key="d")
# the model's up layers carry BN + ReLU (EPI=0: no epilogue)
ep = None if os.environ.get("EPI", "1") == "0" else {
    "scale": torch.rand(96, device="cuda") + 0.5, "shift": torch.rand(96, device="cuda") - 0.5,
    "relu": True}
for _ in range(5):
    sc.inverse_conv_forward(d, wu, spec, cache, None, opts, epilogue=ep)
torch.cuda.synchronize()
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    sc.inverse_conv_forward(d, wu, spec, cache, None, opts, epilogue=ep)
e.record()
torch.cuda.synchronize()
print(f"up 96->96 L1->L0 ({n} rows): {a.elapsed_time(e) / 20:.4f} ms  scatter={os.environ.get('SCB_UPSCATTER', '1')} epi={ep is not None} L1_reorder={os.environ.get('L1_REORDER', '0')}")
