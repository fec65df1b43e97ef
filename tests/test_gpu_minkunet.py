"""Whole-network parity: the MinkUNet bench graph on the B200 engine vs the
same graph on the CPU oracle, on a cropped raycast scan (FP16 storage), and
batch packing is equivalent to separate scans."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _crop(scan, frac):
    c, f, b = scan
    keep = f[:, 0] ** 2 + f[:, 1] ** 2 < (frac * 80.0) ** 2  # disc around the sensor
    return c[keep], f[keep], b


@pytest.fixture(scope="module")
def scan():
    from paper_2204_10319_b200 import workloads
    return _crop(workloads.semantickitti_scan(0), 0.25)


@pytest.mark.parametrize("width,dataflow", [(0.5, "staged"), (1.0, "staged"), (0.5, "auto"),
                                            (1.0, "auto")])
def test_minkunet_matches_oracle(scan, width, dataflow):
    import paper_2204_10319_b200 as sc
    from oracle import sparseconv_oracle as O
    from paper_2204_10319_b200.minkunet import EngineMinkUNet
    from oracle.models import minkunet_oracle as forward_oracle
    coords, feats, boundary = scan
    assert coords.shape[0] > 5000
    model = EngineMinkUNet(width, 4, 0)
    t = sc.quantize_features(sc.SparseTensor(coords, feats, 1, boundary, 1),
                             sc.PrecisionMode.FP16_STORAGE)
    out = model.forward(t, sc.ExecOptions(dataflow=dataflow, index_kind="hash"))
    oc, of, ob = forward_oracle(model.params, width, coords, O.quantize(feats, "fp16"), boundary)
    np.testing.assert_array_equal(out.coords_numpy(), oc)
    got = out.features_numpy().astype(np.float64)
    rel = np.linalg.norm(got - of) / np.linalg.norm(of.astype(np.float64))
    assert rel <= 1e-2, rel


def test_packed_batch_equals_separate(scan):
    """Packing scans along the batch column with a shared boundary is
    bit-identical to running them one by one."""
    import paper_2204_10319_b200 as sc
    from paper_2204_10319_b200.minkunet import EngineMinkUNet
    c0, f0, b0 = scan
    c1, f1 = c0[::2].copy(), f0[::2].copy()
    bnd = b0
    model = EngineMinkUNet(0.5, 4, 1)
    outs = []
    for c, f in ((c0, f0), (c1, f1)):
        t = sc.quantize_features(sc.SparseTensor(c, f, 1, bnd, 1), sc.PrecisionMode.FP16_STORAGE)
        outs.append(model.forward(t).features_numpy())
    pc = np.concatenate([c0, np.concatenate([np.ones((c1.shape[0], 1), np.int64), c1[:, 1:]], 1)])
    pf = np.concatenate([f0, f1])
    t = sc.quantize_features(sc.SparseTensor(pc, pf, 1, bnd, 2), sc.PrecisionMode.FP16_STORAGE)
    packed = model.forward(t)
    pcn = packed.coords_numpy()
    pfn = packed.features_numpy()
    np.testing.assert_array_equal(pfn[pcn[:, 0] == 0], outs[0])
    np.testing.assert_array_equal(pfn[pcn[:, 0] == 1], outs[1])


def test_prefetched_pyramid_is_identical(scan):
    """model.prefetch(t_next) before forward(t) (the serving loop's pipelining
    of the coordinate pyramid) changes nothing: both outputs are bit-identical
    to plain forwards."""
    import paper_2204_10319_b200 as sc
    from paper_2204_10319_b200 import workloads
    from paper_2204_10319_b200.minkunet import EngineMinkUNet
    model = EngineMinkUNet(0.5, 4, 0)
    opts = sc.ExecOptions(dataflow="auto", index_kind="hash")
    c2, f2, b2 = _crop(workloads.semantickitti_scan(1), 0.25)

    def tensor(c, f, b):
        return sc.quantize_features(sc.SparseTensor(c, f, 1, b, 1), sc.PrecisionMode.FP16_STORAGE)

    ref1 = model.forward(tensor(*scan), opts).features_numpy()
    ref2 = model.forward(tensor(c2, f2, b2), opts)
    t1, t2 = tensor(*scan), tensor(c2, f2, b2)
    model.prefetch(t1, opts)
    model.prefetch(t2, opts)
    o1 = model.forward(t1, opts)
    o2 = model.forward(t2, opts)
    np.testing.assert_array_equal(o1.features_numpy(), ref1)
    np.testing.assert_array_equal(o2.coords_numpy(), ref2.coords_numpy())
    np.testing.assert_array_equal(o2.features_numpy(), ref2.features_numpy())


def test_serving_loop_prefetch_overlap(scan):
    """The bench's serving loop: forward(batch i), then upload + prefetch
    batch i+1 on the mapping streams (beside batch i's convolutions), with
    the host running ahead (no synchronisation) over alternating inputs:
    every output equals a plain, synchronised forward of the same input."""
    import torch
    import paper_2204_10319_b200 as sc
    from paper_2204_10319_b200 import workloads
    from paper_2204_10319_b200.minkunet import EngineMinkUNet
    model = EngineMinkUNet(0.5, 4, 0)
    opts = sc.ExecOptions(dataflow="auto", index_kind="hash")
    inputs = [scan, _crop(workloads.semantickitti_scan(1), 0.25),
              _crop(workloads.semantickitti_scan(2), 0.5)]

    def tensor(c, f, b):
        return sc.quantize_features(sc.SparseTensor(c, f, 1, b, 1), sc.PrecisionMode.FP16_STORAGE)

    refs = []
    for c, f, b in inputs:
        o = model.forward(tensor(c, f, b), opts)
        refs.append((o.coords_numpy(), o.features_numpy()))
    outs, order = [], [0, 1, 2, 1, 0, 2, 2, 1]
    t = tensor(*inputs[order[0]])
    for i, j in enumerate(order):
        o = model.forward(t, opts)
        outs.append((j, o))
        if i + 1 < len(order):
            t = tensor(*inputs[order[i + 1]])
            ev = torch.cuda.current_stream().record_event()
            model.prefetch(t, opts, coords_ready=ev)
    for j, o in outs:
        np.testing.assert_array_equal(o.coords_numpy(), refs[j][0])
        np.testing.assert_array_equal(o.features_numpy(), refs[j][1])
