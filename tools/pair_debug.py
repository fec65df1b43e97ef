"""Where does the CTA-pair kernel differ from the single-CTA kernel (debug)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10319_b200 as sc  # noqa: E402
from paper_2204_10319_b200 import workloads  # noqa: E402
from paper_2204_10319_b200.mapping import reorder_by_presence  # noqa: E402

rng = np.random.default_rng(0)
c, _, b = workloads.semantickitti_scan(4)
t = sc.SparseTensor(c, np.zeros((c.shape[0], 1), np.float32), 1, b, 1)
p = reorder_by_presence(t.coordset, 3, "hash")
n = p.num_points
for cin, cout in ((96, 96), (32, 96), (96, 32), (64, 96), (96, 64), (128, 128), (48, 48)):
    x = sc.SparseTensor._wrap(torch.from_numpy(rng.standard_normal((n, cin)).astype(np.float16)).cuda(),
                              1, b, 1, p)
    w = sc.WeightTensor(rng.normal(0, 1 / np.sqrt(27 * cin), (27, cin, cout)).astype(np.float32), 3, 3)
    spec = sc.LayerSpec(3, 1, cin, cout)
    res = {}
    for shape in ((2, 0), (4, 0)):
        o = sc.ExecOptions(dataflow="fused", index_kind="hash", layer_label="L", kernel_shapes={"L": shape})
        res[shape] = sc.sparse_conv_forward(x, w, spec, None, None, o).features.float().cpu().numpy()
    a, g = res[(2, 0)], res[(4, 0)]
    a16, g16 = a.astype(np.float16), g.astype(np.float16)
    ulp = np.abs(np.spacing(a16).astype(np.float32))
    du = np.abs(a - g) / np.maximum(ulp, 2.0 ** -24)
    rel = np.linalg.norm(a - g) / np.linalg.norm(a)
    print(f"  max ulps {du.max():.1f}, elems >1ulp {(du > 1).sum()}, >0 {(du > 0).sum()} of {a.size}, rel L2 {rel:.3g}; worst at value {a.flat[du.argmax()]:.4g} vs {g.flat[du.argmax()]:.4g}")
    bad = np.abs(a - g) > 1e-3 * (1 + np.abs(a))
    rows = np.nonzero(bad.any(1))[0]
    cols = np.nonzero(bad.any(0))[0]
    print(f"{cin}->{cout}: bad elems {bad.sum()} rows {rows.size} cols {cols.size} "
          f"maxdiff {np.abs(a - g).max():.4g}; rows%256<128 frac "
          f"{np.mean((rows % 256) < 128) if rows.size else 0:.2f}; cols {cols[:8]}..{cols[-8:] if cols.size else ''}; "
          f"tiles {np.unique(rows // 128)[:10]}", flush=True)
