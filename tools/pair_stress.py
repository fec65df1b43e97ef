"""Stress: the CTA-pair kernel vs the single-CTA kernel on the same layer,
repeated with the allocator state shuffled in between (debug tool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10319_b200 as sc  # noqa: E402
from paper_2204_10319_b200 import workloads  # noqa: E402
from paper_2204_10319_b200.core import CoordinateSet  # noqa: E402
from paper_2204_10319_b200.mapping import reorder_by_presence  # noqa: E402

rng = np.random.default_rng(0)
c, _, b = workloads.semantickitti_scan(4)
t0 = sc.SparseTensor(c, np.zeros((c.shape[0], 1), np.float32), 1, b, 1)
p = reorder_by_presence(t0.coordset, 3, "hash")
n = p.num_points
tiles = n // 128 - 1
tiles -= 1 - tiles % 2
keep = (tiles - 1) * 128 + 37
cs = reorder_by_presence(CoordinateSet(p.coords[:keep].clone(), b, 1), 3, "hash")
a = torch.from_numpy(rng.standard_normal((keep, 64)).astype(np.float16)).cuda()
bb = torch.from_numpy(rng.standard_normal((keep, 32)).astype(np.float16)).cuda()
res = torch.from_numpy(rng.standard_normal((keep, 96)).astype(np.float16)).cuda()
x = sc.SparseTensor._wrap(a, 1, b, 1, cs)
w = sc.WeightTensor(rng.normal(0, 0.05, (27, 96, 96)).astype(np.float32), 3, 3)
ep = {"scale": torch.from_numpy(rng.uniform(0.8, 1.2, 96).astype(np.float32)).cuda(),
      "shift": torch.from_numpy(rng.normal(0, 0.05, 96).astype(np.float32)).cuda(),
      "residual": res, "relu": True}
spec = sc.LayerSpec(3, 1, 96, 96)


def run(shape):
    o = sc.ExecOptions(dataflow="fused", index_kind="hash", layer_label="L", kernel_shapes={"L": shape})
    return sc.sparse_conv_forward(x, w, spec, None, None, o, epilogue=ep, concat=bb).features.float()


want = run((2, 0))
bad = 0
junk = []
for it in range(int(os.environ.get("ITERS", "60"))):
    junk.append(torch.randn(int(rng.integers(1, 64)) << 16, device="cuda"))
    if len(junk) > 8:
        junk.pop(int(rng.integers(0, len(junk))))
    shape = [(4, 0), (5, 0), (2, 0), (1, 0)][it % 4]
    got = run(shape)
    d = (got - want).abs()
    if float(d.max()) > 1e-2:
        bad += 1
        rows = torch.nonzero(d > 1e-2)[:, 0]
        print(f"it {it} shape {shape}: max {float(d.max()):.4g}, bad elems {int((d > 1e-2).sum())}, "
              f"tiles {sorted(set((rows // 128).tolist()))[:12]}, n_tiles {(keep + 127) // 128}", flush=True)
print("bad", bad)
