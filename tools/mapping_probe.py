"""Time the level-0 mapping kernels of the bench's 8-scan pack as the model
runs them: presence relabelling (scb_presence_masks + scb_mask_sort + the
relabelled index) and the masked k3 map search.  SCB_LIB_NAME picks a build
for A/B."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10319_b200 as sc  # noqa: E402
from paper_2204_10319_b200.mapping import map_search_masked, reorder_by_presence  # noqa: E402
from bench import load_scans, pack  # noqa: E402

c, f, b = pack(load_scans(range(8)))
ct = torch.from_numpy(c.astype(np.int32)).cuda()
off = sc.enumerate_offsets(3, 3)


def relabel():
    t0 = sc.SparseTensor(ct, np.zeros((c.shape[0], 1), np.float32), 1, b, 8)
    return reorder_by_presence(t0.coordset, 3, "hash")


def search(p):
    idx = sc.build_index(p, "hash")
    return map_search_masked(idx, p, off, p.derived[("presence", 3)])


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return a.elapsed_time(e) / reps


p = relabel()
print(f"lib={os.environ.get('SCB_LIB_NAME', 'default')} relabel {timed(relabel):.4f} ms  "
      f"index+masked search {timed(lambda: search(p)):.4f} ms  ({c.shape[0]} rows)")
