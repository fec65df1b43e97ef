"""``SparseConv3d``: the module form north_star names (kernel_size, stride,
dilation, transposed) over the drop-in operator API.

The reference has no module class (its layers are
``LayerSpec`` + ``WeightTensor`` passed to ``sparse_conv_forward`` /
``inverse_conv_forward``, execution.py:450-551); this is that pair held
together, with TorchSparse's constructor arguments.  ``dilation`` is a B200
extension (the reference's windows are dense cubes, core.py:150-161): the
window's offsets are scaled by it (scb_map_search_dilated), supported for
stride-1 layers.  A transposed layer replays the map of the strided layer
whose ``reuse_key`` it names, from the ``map_cache`` both are called with
(the reference's CachedMap protocol, execution.py:126-134)."""

from __future__ import annotations

import numpy as np
import torch

from .core import SparseTensor, WeightTensor
from .execution import ExecOptions, LayerSpec, inverse_conv_forward, sparse_conv_forward


class SparseConv3d:
    """y = conv(x) (+ bias) over a sparse tensor.

    Weights are ``(K^3, C_in, C_out)`` f32, initialised N(0, 1/sqrt(K^3 C_in))
    like reference network.py:183-193 unless ``weight`` is given."""

    def __init__(self, in_channels: int, out_channels: int, kernel_size: int = 3,
                 stride: int = 1, dilation: int = 1, bias: bool = False,
                 transposed: bool = False, reuse_key: str | None = None, weight=None,
                 seed: int = 0, index_kind: str | None = None):
        vol = kernel_size ** 3
        if weight is None:
            rng = np.random.default_rng(seed)
            weight = rng.normal(0.0, 1.0 / np.sqrt(vol * in_channels),
                                (vol, in_channels, out_channels)).astype(np.float32)
        self.weight = WeightTensor(np.asarray(weight, np.float32), kernel_size, 3)
        self.transposed = bool(transposed)
        if transposed and stride != 1 and reuse_key is None:
            raise ValueError("a transposed layer names the strided layer it inverts (reuse_key)")
        if stride > 1 and not transposed and reuse_key is None:
            reuse_key = f"conv{id(self)}"   # so a transposed layer can refer to this map
        self.spec = LayerSpec(kernel_size, 1 if transposed else stride, in_channels,
                              out_channels, transposed=self.transposed, reuse_key=reuse_key,
                              index_kind=index_kind, dilation=dilation)
        self.bias = torch.zeros(out_channels, dtype=torch.float32, device="cuda") if bias else None

    @property
    def reuse_key(self):
        return self.spec.reuse_key

    def __call__(self, x: SparseTensor, map_cache: dict | None = None,
                 options: ExecOptions | None = None) -> SparseTensor:
        return self.forward(x, map_cache, options)

    def forward(self, x: SparseTensor, map_cache: dict | None = None,
                options: ExecOptions | None = None) -> SparseTensor:
        ep = {"bias": self.bias} if self.bias is not None else None
        if self.transposed:
            if map_cache is None:
                raise ValueError("a transposed layer needs the map_cache of its strided layer")
            return inverse_conv_forward(x, self.weight, self.spec, map_cache, None, options,
                                        epilogue=ep)
        return sparse_conv_forward(x, self.weight, self.spec, None, map_cache, options,
                                   epilogue=ep)
