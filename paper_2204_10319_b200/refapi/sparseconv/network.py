"""``sparseconv.network`` on the B200 engine (reference ``network.py``):
the same JSON schema and bit-identical parameters (``Network.build``); the
forward runs every layer on the engine and returns a host tensor."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2204_10319_b200 import network as _eng

from .core import SparseTensor, _engine_tensor, _wrap_result

POINTWISE_KINDS = _eng.POINTWISE_KINDS
CONV_KINDS = _eng.CONV_KINDS
ConfigError = _eng.ConfigError
LayerConfig = _eng.LayerConfig
NetworkConfig = _eng.NetworkConfig
load_builtin_config = _eng.load_builtin_config


def load_network_config(spec: str) -> NetworkConfig:
    """A file path (``*.json``) or a builtin name (reference network.py:166-171)."""
    if str(spec).endswith(".json"):
        return NetworkConfig.from_file(spec)
    return load_builtin_config(str(spec))


@dataclass
class Network(_eng.Network):
    """A configured network with materialised parameters (reference
    network.py:174-278)."""

    @staticmethod
    def build(config: NetworkConfig, spatial_dims: int = 3) -> "Network":
        eng = _eng.Network.build(config, spatial_dims)
        return Network(eng.config, eng.weights, eng.pointwise)

    def describe(self) -> list[dict]:
        """Structural layer descriptions as plain data (reference
        network.py:218-232)."""
        out = []
        for L in self.config.layers:
            entry: dict = {"id": L.layer_id, "kind": L.kind}
            if L.kind in CONV_KINDS:
                entry.update(kernel_size=L.kernel_size, stride=L.stride,
                             weights=np.asarray(self.weights[L.layer_id].weights))
                if L.kind == "inverse_conv":
                    entry["reuse"] = L.reuse
            else:
                entry.update(self.pointwise.get(L.layer_id, {}))
            out.append(entry)
        return out

    def forward(self, t: SparseTensor, strategies: dict | None = None, options=None
                ) -> SparseTensor:
        """The whole network on the device; one host copy of the result."""
        return _wrap_result(super().forward(_engine_tensor(t), strategies, options))
