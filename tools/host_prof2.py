"""Host-side profile of EngineMinkUNet.forward in the serving loop (cProfile)."""
import cProfile
import os
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10319_b200 as sc  # noqa: E402
from paper_2204_10319_b200.minkunet import EngineMinkUNet  # noqa: E402
from bench import load_scans, pack, DEFAULT_STRATEGY  # noqa: E402

c, f, b = pack(load_scans(range(8)))
model = EngineMinkUNet(1.0, 4, 0, strategy=str(DEFAULT_STRATEGY))
cd = torch.from_numpy(c.astype(np.int32)).cuda()
fd = torch.from_numpy(f).cuda()
ev = torch.cuda.Event()
ev.record()
opts = sc.ExecOptions(index_kind="hash", dataflow="auto")


def mk():
    return sc.quantize_features(sc.SparseTensor(cd, fd, 1, b, 8, validate=False),
                                sc.PrecisionMode.FP16_STORAGE)


nxt = mk()
model.prefetch(nxt, opts, coords_ready=ev)
for _ in range(30):
    t = nxt
    model.forward(t, opts)
    nxt = mk()
    model.prefetch(nxt, opts, coords_ready=ev)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    t = nxt
    model.forward(t, opts)
    nxt = mk()
    model.prefetch(nxt, opts, coords_ready=ev)
pr.disable()
torch.cuda.synchronize()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
