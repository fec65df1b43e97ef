"""CPU oracle for the sparse-convolution forward path — TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference package
``sparseconv`` (``/root/reference/pkg/src/sparseconv``; citations below are
``file:line`` relative to that directory).  It exists to *check* the B200
engine, never to run inside it: only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import it.
The product package ``paper_2204_10319_b200`` never imports this file and has
no CPU fallback.

Parity of this oracle with the reference is pinned by golden vectors that
were produced by importing the unmodified reference
(``tests/golden/make_golden.py`` → ``tests/golden/*.npz``) and checked by
``tests/test_oracle_golden.py``.

Numerics contract restated here:
  * gather copies storage-dtype rows            (execution.py:159-180)
  * each offset's matmul: storage rows -> f32, times f32 weights, f32 out
                                                (execution.py:356-367)
  * scatter folds f64 in ascending buffer-row order, rounded once to f32
                                                (kernels.py:38-50)
  * the f32 centre GEMM is added after that rounding (execution.py:423-428)
  * the layer output is cast to the storage dtype (execution.py:506)
"""

from __future__ import annotations

from itertools import product

import numpy as np

MISS = -1


# ---------------------------------------------------------------- keys / offsets

def flatten(coords, boundary, batch_size=1):
    """Batch-major flat key ``((b*bx + x)*by + y)*bz + z`` (core.py:46-66)."""
    total = int(batch_size)
    for b in boundary:
        if int(b) <= 0:
            raise ValueError("boundary extents must be positive")
        total *= int(b)
    if total >= 1 << 62:
        raise ValueError("coordinate space too large to key into int64")
    c = np.asarray(coords, dtype=np.int64)
    key = c[:, 0].copy()
    for d, b in enumerate(boundary):
        key = key * int(b) + c[:, d + 1]
    return key


def unflatten(keys, boundary):
    """Inverse of :func:`flatten` (core.py:69-79)."""
    keys = np.asarray(keys, dtype=np.int64)
    out = np.empty((keys.shape[0], 1 + len(boundary)), dtype=np.int64)
    rest = keys.copy()
    for d in reversed(range(len(boundary))):
        out[:, d + 1] = rest % int(boundary[d])
        rest //= int(boundary[d])
    out[:, 0] = rest
    return out


def voxelize(points, voxel_size, reduce="mean", spatial_dims=3):
    """core.py:174-216: cells = floor((p - min) / voxel_size) in f64, boundary
    = max + 1, rows sorted by flat key; duplicates merged by the f64 mean
    (np.bincount: sequential sum in point order, core.py:207-211) or the
    first point (core.py:205-206).  Returns (coords int64, features f32,
    boundary)."""
    pts = np.asarray(points, dtype=np.float64)
    xyz, feats = pts[:, :spatial_dims], pts[:, spatial_dims:]
    cells = np.floor((xyz - xyz.min(axis=0)) / voxel_size).astype(np.int64)
    boundary = tuple(int(m) + 1 for m in cells.max(axis=0))
    key = np.zeros(cells.shape[0], dtype=np.int64)
    for d, b in enumerate(boundary):
        key = key * b + cells[:, d]
    uniq, first, inverse = np.unique(key, return_index=True, return_inverse=True)
    if reduce == "first":
        merged = feats[first].astype(np.float32)
    else:
        counts = np.bincount(inverse, minlength=uniq.shape[0]).astype(np.float64)
        merged = np.empty((uniq.shape[0], feats.shape[1]), dtype=np.float32)
        for c in range(feats.shape[1]):
            merged[:, c] = (np.bincount(inverse, weights=feats[:, c], minlength=uniq.shape[0])
                            / counts).astype(np.float32)
    return np.concatenate([np.zeros((uniq.shape[0], 1), np.int64),
                           unflatten(uniq, boundary)[:, 1:]], axis=1), merged, boundary


def offsets(dim, kernel_size):
    """Lexicographic K**D window; centred for odd K, {0..K-1} for even K
    (mapping.py:63-79, EVEN_KERNEL_OFFSET_BASE = 0 at mapping.py:26)."""
    lo = -((kernel_size - 1) // 2) if kernel_size % 2 == 1 else 0
    axis = list(range(lo, lo + kernel_size))
    return np.array(list(product(axis, repeat=dim)), dtype=np.int64).reshape(-1, dim)


def center_of(kernel_size, dim):
    """Index of the zero offset, or None for even K (mapping.py:55-60)."""
    return (kernel_size ** dim - 1) // 2 if kernel_size % 2 == 1 else None


def downsample_boundary(boundary, stride):
    """ceil(b / s) per dimension (mapping.py:211-213)."""
    return tuple(-(-int(b) // stride) for b in boundary)


# ---------------------------------------------------------------- coordinates

def output_coords(in_coords, kernel_size, stride, out_boundary, batch_size=1):
    """Active outputs of a layer (mapping.py:216-248).

    stride 1 keeps the input rows as-is.  Otherwise every input p proposes
    u = p - delta for each offset, kept iff u % s == 0, u >= 0 and
    u < s * b_out in every dimension; the survivors u // s are deduplicated
    and returned in ascending flat-key order.
    """
    c = np.asarray(in_coords, dtype=np.int64)
    if stride == 1:
        return c
    dim = c.shape[1] - 1
    off = offsets(dim, kernel_size)
    hi = stride * np.asarray(out_boundary, dtype=np.int64)
    keys = []
    for n in range(off.shape[0]):
        u = c[:, 1:] - off[n]
        ok = ((u % stride) == 0).all(1) & (u >= 0).all(1) & (u < hi).all(1)
        if ok.any():
            cand = np.concatenate([c[ok, :1], u[ok] // stride], axis=1)
            keys.append(flatten(cand, out_boundary, batch_size))
    if not keys:
        return np.empty((0, 1 + dim), dtype=np.int64)
    return unflatten(np.unique(np.concatenate(keys)), out_boundary)


# ---------------------------------------------------------------- kernel map

def _lookup(sorted_keys, order, in_boundary, batch_size, probe):
    """Row of each probe coordinate in the input set, MISS when absent or
    out of bounds (the observable contract of GridIndex/HashIndex.query,
    mapping.py:106-119 and 166-189)."""
    res = np.full(probe.shape[0], MISS, dtype=np.int64)
    bnd = np.asarray(in_boundary, dtype=np.int64)
    ok = (probe[:, 0] >= 0) & (probe[:, 0] < batch_size) \
        & (probe[:, 1:] >= 0).all(1) & (probe[:, 1:] < bnd).all(1)
    if not ok.any() or sorted_keys.shape[0] == 0:
        return res
    k = flatten(probe[ok], in_boundary, batch_size)
    pos = np.searchsorted(sorted_keys, k)
    pos_c = np.minimum(pos, sorted_keys.shape[0] - 1)
    hit = sorted_keys[pos_c] == k
    rows = np.where(hit, order[pos_c], MISS)
    res[np.nonzero(ok)[0]] = rows
    return res


def kernel_map(in_coords, in_boundary, out_coords, kernel_size, stride,
               batch_size=1, use_symmetry=None, dilation=1):
    """Per-offset (j, k) pairs with p_j == s*q_k + delta_n, rows sorted by k
    (mapping.py:289-319); stride-1 odd-K maps derive the upper half from the
    lower half (mapping.py:322-339).  Returns a list of (m_n, 2) int64."""
    cin = np.asarray(in_coords, dtype=np.int64)
    cout = np.asarray(out_coords, dtype=np.int64)
    dim = cin.shape[1] - 1
    off = offsets(dim, kernel_size)
    volume = off.shape[0]
    center = center_of(kernel_size, dim)
    if use_symmetry is None:
        use_symmetry = stride == 1 and center is not None and volume > 1
    keys = flatten(cin, in_boundary, batch_size) if cin.shape[0] else np.empty(0, np.int64)
    order = np.argsort(keys, kind="stable")
    sorted_keys = keys[order]
    searched = range(center + 1) if use_symmetry else range(volume)
    pairs = [np.empty((0, 2), dtype=np.int64) for _ in range(volume)]
    for n in searched:
        probe = cout.copy()
        probe[:, 1:] = stride * cout[:, 1:] + dilation * off[n]   # dilation: B200 extension
        j = _lookup(sorted_keys, order, in_boundary, batch_size, probe)
        k = np.nonzero(j != MISS)[0]
        pairs[n] = np.stack([j[k], k], axis=1).astype(np.int64)
    if use_symmetry:
        for n in range(center):
            mirrored = pairs[n][:, ::-1]
            pairs[volume - 1 - n] = np.ascontiguousarray(
                mirrored[np.argsort(mirrored[:, 1], kind="stable")])
    return pairs


def swap_roles(pairs):
    """Inverse-layer map: (j, k) -> (k, j), re-sorted by the new output row
    (mapping.py:277-286)."""
    out = []
    for p in pairs:
        q = p[:, ::-1]
        out.append(np.ascontiguousarray(q[np.argsort(q[:, 1], kind="stable")]))
    return out


# ---------------------------------------------------------------- plan

def plan(pairs, n_in, n_out, skip_center=None):
    """Offset-major buffer layout plus both stationary CSR indexes
    (mapping.py:377-418).  ``skip_center`` is the centre offset index to
    leave out (zero-width slice) or None."""
    sizes = np.array([p.shape[0] for p in pairs], dtype=np.int64)
    if skip_center is not None:
        sizes[skip_center] = 0
    starts = np.zeros(len(pairs) + 1, dtype=np.int64)
    np.cumsum(sizes, out=starts[1:])
    kept = [p for n, p in enumerate(pairs) if n != skip_center and p.shape[0]]
    stacked = np.concatenate(kept, 0) if kept else np.empty((0, 2), np.int64)
    row_input = np.ascontiguousarray(stacked[:, 0])
    row_output = np.ascontiguousarray(stacked[:, 1])
    in_indptr = np.zeros(n_in + 1, dtype=np.int64)
    np.cumsum(np.bincount(row_input, minlength=n_in), out=in_indptr[1:])
    out_indptr = np.zeros(n_out + 1, dtype=np.int64)
    np.cumsum(np.bincount(row_output, minlength=n_out), out=out_indptr[1:])
    return {
        "buffer_offsets": starts,
        "row_input": row_input,
        "row_output": row_output,
        "in_indptr": in_indptr,
        "in_rows": np.argsort(row_input, kind="stable").astype(np.int64),
        "out_indptr": out_indptr,
        "out_rows": np.argsort(row_output, kind="stable").astype(np.int64),
        "total": int(starts[-1]),
    }


# ---------------------------------------------------------------- movement

def gather(features, pl):
    """Buffer row r = features[row_input[r]], storage dtype kept
    (execution.py:159-180; all traversal orders are bit-identical)."""
    return np.asarray(features)[pl["row_input"]]


def scatter(buffer, pl, n_out):
    """out[k] = f32(sum over buffer rows of k, ascending, in f64)
    (execution.py:183-218, kernels.py:38-50)."""
    buffer = np.asarray(buffer)
    out = np.empty((n_out, buffer.shape[1]), dtype=np.float32)
    if pl["total"] == 0:
        out[:] = 0
        return out
    for c in range(buffer.shape[1]):
        out[:, c] = np.bincount(pl["row_output"], weights=buffer[:, c].astype(np.float64),
                                minlength=n_out)
    return out


# ---------------------------------------------------------------- grouping (host)

def partition(sizes, eps, schedule):
    """Alg. 3 greedy left-to-right grouping (execution.py:221-247)."""
    if not 0.0 <= eps <= 1.0:
        raise ValueError("eps must lie in [0, 1]")
    sizes = np.asarray(sizes, dtype=np.int64)
    schedule = list(schedule)
    out, i = [], 0
    while i < len(schedule):
        lo = hi = int(sizes[schedule[i]])
        start = i
        i += 1
        while i < len(schedule):
            n = int(sizes[schedule[i]])
            nlo, nhi = min(lo, n), max(hi, n)
            if (0.0 if nhi == 0 else 1.0 - nlo / nhi) > eps:
                break
            lo, hi = nlo, nhi
            i += 1
        out.append((start, i))
    return out


def groups(sizes, eps, threshold, schedule, symmetric):
    """(start, end, mode, padded_rows) per group (execution.py:309-328)."""
    sizes = np.asarray(sizes, dtype=np.int64)
    volume = sizes.shape[0]
    res = []
    for s, e in partition(sizes, eps, schedule):
        mem = list(schedule[s:e])
        if symmetric:
            mem += [volume - 1 - n for n in mem]
        top = max((int(sizes[m]) for m in mem), default=0)
        if top < threshold:
            res.append((s, e, "batched", sum(top - int(sizes[m]) for m in mem)))
        else:
            res.append((s, e, "sequential", 0))
    return res


def schedule_of(volume, center, stride):
    """First half without centre + mirrors for stride-1 odd K, else all
    offsets (execution.py:296-306)."""
    if stride == 1 and center is not None and volume > 1:
        return list(range(center)), True
    return list(range(volume)), False


# ---------------------------------------------------------------- GEMM

def offset_matmuls(buffer, weights, pl):
    """f32 partials for every buffer slice: storage -> f32 times f32 weights
    (execution.py:331-368; grouping changes only the batching, so per-offset
    matmuls give the same rows up to BLAS summation order)."""
    w = np.asarray(weights, dtype=np.float32)
    out = np.zeros((pl["total"], w.shape[2]), dtype=np.float32)
    st = pl["buffer_offsets"]
    for n in range(st.shape[0] - 1):
        if st[n + 1] > st[n]:
            out[st[n]:st[n + 1]] = np.asarray(buffer[st[n]:st[n + 1]], np.float32) @ w[n]
    return out


# ---------------------------------------------------------------- layers

def quantize(features, precision):
    """fp16 round-to-nearest with saturation to +-65504 (core.py:219-238)."""
    f = np.asarray(features)
    if precision == "fp32":
        return f.astype(np.float32)
    with np.errstate(over="ignore"):
        q = f.astype(np.float16)
    bad = np.isinf(q) & np.isfinite(f)
    if bad.any():
        q = q.copy()
        q[bad] = (np.sign(f[bad]) * 65504.0).astype(np.float16)
    return q


def conv_forward(coords, features, boundary, weights, kernel_size, stride,
                 batch_size=1, return_map=False, dilation=1):
    """One sparse conv layer (execution.py:450-509).

    Returns (out_coords, out_features[storage dtype], out_boundary) and, with
    ``return_map``, also the kernel map pairs for inverse layers."""
    coords = np.asarray(coords, dtype=np.int64)
    features = np.asarray(features)
    storage = features.dtype
    w = np.asarray(weights, dtype=np.float32)
    if kernel_size == 1 and stride == 1:
        out = features.astype(np.float32) @ w[0]
        res = (coords, out.astype(storage), tuple(boundary))
        return res + (None,) if return_map else res
    dim = coords.shape[1] - 1
    if stride == 1:
        out_coords, out_boundary = coords, tuple(boundary)
    else:
        out_boundary = downsample_boundary(boundary, stride)
        out_coords = output_coords(coords, kernel_size, stride, out_boundary, batch_size)
    pairs = kernel_map(coords, boundary, out_coords, kernel_size, stride, batch_size,
                       dilation=dilation)
    center = center_of(kernel_size, dim)
    skip = center if stride == 1 else None
    pl = plan(pairs, coords.shape[0], out_coords.shape[0], skip)
    partial = offset_matmuls(gather(features, pl), w, pl)
    out = scatter(partial, pl, out_coords.shape[0])
    if skip is not None:
        out += features.astype(np.float32) @ w[center]
    res = (out_coords, out.astype(storage), out_boundary)
    return res + (pairs,) if return_map else res


def inverse_forward(features, weights, cached_pairs, n_in_fine):
    """Transposed layer replaying a strided map with roles swapped
    (execution.py:512-551).  Output rows are the cached layer's inputs."""
    features = np.asarray(features)
    storage = features.dtype
    sw = swap_roles(cached_pairs)
    pl = plan(sw, features.shape[0], n_in_fine, None)
    partial = offset_matmuls(gather(features, pl), weights, pl)
    return scatter(partial, pl, n_in_fine).astype(storage)


def pointwise(features, op, bias=None, scale=None, shift=None):
    """relu / bias_add / bn_fold, f32 compute cast back (execution.py:554-576)."""
    f = np.asarray(features)
    st = f.dtype
    if op == "relu":
        return np.maximum(f, 0)
    if op == "bias_add":
        return (f.astype(np.float32) + np.asarray(bias, np.float32)).astype(st)
    if op == "bn_fold":
        return (f.astype(np.float32) * np.asarray(scale, np.float32)
                + np.asarray(shift, np.float32)).astype(st)
    raise ValueError(f"unknown pointwise op {op!r}")


# ---------------------------------------------------------------- network

def build_params(doc, spatial_dims=3):
    """Deterministic parameters in layer order from ``param_seed``
    (network.py:181-201)."""
    rng = np.random.default_rng(int(doc.get("param_seed", 0)))
    ch = int(doc["in_channels"])
    weights, pw = {}, {}
    for i, L in enumerate(doc["layers"]):
        kind = L["kind"]
        lid = str(L.get("id") or f"{kind}_{i}")
        if kind in ("conv", "inverse_conv"):
            vol = int(L.get("kernel_size", 1)) ** spatial_dims
            w = rng.normal(0.0, 1.0 / np.sqrt(vol * ch), size=(vol, ch, int(L["out_channels"])))
            weights[lid] = w.astype(np.float32)
            ch = int(L["out_channels"])
        elif kind == "bias_add":
            pw[lid] = {"bias": rng.normal(0.0, 0.1, size=ch).astype(np.float32)}
        elif kind == "bn_fold":
            pw[lid] = {"scale": rng.uniform(0.8, 1.2, size=ch).astype(np.float32),
                       "shift": rng.normal(0.0, 0.05, size=ch).astype(np.float32)}
    return weights, pw


def network_forward(doc, coords, features, boundary, batch_size=1, params=None):
    """Whole-network forward over the reference JSON schema
    (network.py:250-278).  Returns (coords, features)."""
    weights, pw = params if params is not None else build_params(doc, coords.shape[1] - 1)
    feats = quantize(features, doc.get("precision", "fp32"))
    coords = np.asarray(coords, dtype=np.int64)
    boundary = tuple(boundary)
    cache = {}
    for i, L in enumerate(doc["layers"]):
        kind = L["kind"]
        lid = str(L.get("id") or f"{kind}_{i}")
        if kind == "conv":
            k, s = int(L.get("kernel_size", 1)), int(L.get("stride", 1))
            oc, of, ob, pairs = conv_forward(coords, feats, boundary, weights[lid], k, s,
                                             batch_size, return_map=True)
            if pairs is not None:
                cache[lid] = (pairs, coords, boundary)
            coords, feats, boundary = oc, of, ob
        elif kind == "inverse_conv":
            pairs, fine_coords, fine_boundary = cache[L["reuse"]]
            feats = inverse_forward(feats, weights[lid], pairs, fine_coords.shape[0])
            coords, boundary = fine_coords, fine_boundary
        else:
            feats = pointwise(feats, kind, **pw.get(lid, {}))
    return coords, feats
