"""Stress the CTA-pair kernel inside PDL-chained launch sequences: for each
(C_in, C_out, shape) run chains of layers back to back (pair layers after
single layers, no sync), compare each pair output with the single-CTA
kernel's (debug tool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10319_b200 as sc  # noqa: E402
from paper_2204_10319_b200 import workloads  # noqa: E402
from paper_2204_10319_b200.mapping import reorder_by_presence  # noqa: E402

rng = np.random.default_rng(1)
c, _, b = workloads.semantickitti_scan(4)
t0 = sc.SparseTensor(c, np.zeros((c.shape[0], 1), np.float32), 1, b, 1)
p = reorder_by_presence(t0.coordset, 3, "hash")
n = p.num_points
cfgs = [(32, 32), (64, 64), (96, 96), (128, 128), (64, 96)]
layers = []
for ci, co in cfgs:
    w = sc.WeightTensor(rng.normal(0, 1 / np.sqrt(27 * ci), (27, ci, co)).astype(np.float32), 3, 3)
    f = torch.from_numpy(rng.standard_normal((n, ci)).astype(np.float16)).cuda()
    res = torch.from_numpy(rng.standard_normal((n, co)).astype(np.float16)).cuda()
    ep = {"scale": torch.ones(co, device="cuda"), "shift": torch.zeros(co, device="cuda"),
          "residual": res, "relu": True}
    layers.append((sc.SparseTensor._wrap(f, 1, b, 1, p), w, sc.LayerSpec(3, 1, ci, co), ep))


def run(i, shape):
    x, w, spec, ep = layers[i]
    o = sc.ExecOptions(dataflow="fused", index_kind="hash", layer_label="L", kernel_shapes={"L": shape})
    return sc.sparse_conv_forward(x, w, spec, None, None, o, epilogue=ep).features


want = [run(i, (2, 0)).float() for i in range(len(layers))]
torch.cuda.synchronize()
bad = 0
shapes = [tuple(int(v) for v in x.split(":")) for x in
          os.environ.get("SHAPES", "4:0,5:0,5:48,4:48").split(",")]
for it in range(int(os.environ.get("ITERS", "40"))):
    outs = []
    for i in range(len(layers)):          # chains: single, pair, single, pair ... no sync
        run((i + 1) % len(layers), (2, 0))
        sh = shapes[(it + i) % len(shapes)]
        outs.append((i, sh, run(i, sh)))
    torch.cuda.synchronize()
    for i, sh, o in outs:
        d = (o.float() - want[i]).abs()
        m = float(d.max())
        if m > 2e-2:
            bad += 1
            rows = torch.nonzero(d > 2e-2)[:, 0]
            print(f"it {it} layer {cfgs[i]} shape {sh}: max {m:.4g}, bad {int((d > 2e-2).sum())}, "
                  f"tiles {sorted(set((rows // 128).tolist()))[:8]}", flush=True)
print("bad", bad, "of", int(os.environ.get("ITERS", "40")) * len(layers))
