"""Any-precision layer data contract (reference quantizer.py:27-28, 75-119).

The offline quantizer is out of scope; the hot path only
consumes its output type.  This mirror accepts the same fields and the engine
also accepts the reference's own ``AnyPrecisionLayer`` objects (duck typing on
``n_min``, ``n_max``, ``codes``, ``centroid_tables``, ``shape``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ParameterError, ShapeError

MIN_BITS = 2
MAX_BITS = 8


@dataclass
class AnyPrecisionLayer:
    """Parent-model codes plus one fp16 centroid table per supported bit-width."""

    n_min: int
    n_max: int
    codes: np.ndarray                       # (out_channels, in_features) uint8
    centroid_tables: dict                   # k -> (out_channels, 2**k) float16
    shape: tuple
    channel_sse: dict = field(default_factory=dict)
    level_codes: dict = field(default_factory=dict)

    def __post_init__(self):
        if not MIN_BITS <= self.n_min <= self.n_max <= MAX_BITS:
            raise ParameterError(
                f"bit range [{self.n_min}, {self.n_max}] outside [{MIN_BITS}, {MAX_BITS}]"
            )
        if tuple(self.codes.shape) != tuple(self.shape):
            raise ShapeError("codes shape does not match declared layer shape")
        for k in range(self.n_min, self.n_max + 1):
            if k not in self.centroid_tables:
                raise ParameterError(f"missing centroid table for {k}-bit")

    @property
    def out_channels(self) -> int:
        return self.shape[0]

    @property
    def in_features(self) -> int:
        return self.shape[1]

    def supported_bits(self) -> range:
        return range(self.n_min, self.n_max + 1)

    def codes_at(self, k: int) -> np.ndarray:
        """Top-k-bit codes (quantizer.py:115-119)."""
        if k not in self.supported_bits():
            raise ParameterError(f"bit width {k} not in [{self.n_min}, {self.n_max}]")
        return self.codes >> (self.n_max - k)


def supported_bits(layer) -> range:
    return range(layer.n_min, layer.n_max + 1)
