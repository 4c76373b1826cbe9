"""R-index vocabulary (pkg/src/nbz/rindex.py:24-56, 155-161).

All three variants run on the B200 path: coordinate keys,
velocity keys and the six-field coord+velocity keys (§8 f4); the key
construction and the segmented sort themselves run on device
(csrc/rindex.cu).  ``segment_bounds`` and ``Segment`` keep the reference's
meaning: segment boundaries are derived from (n, segment_size), never stored.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass
from typing import Tuple

import numpy as np

from .errors import ValidationError


class RIndexVariant(enum.Enum):
    COORDINATE = "coord"
    VELOCITY = "vel"
    COORD_VELOCITY = "coordvel"

    @property
    def field_indices(self) -> Tuple[int, ...]:
        if self is RIndexVariant.COORDINATE:
            return (0, 1, 2)
        if self is RIndexVariant.VELOCITY:
            return (3, 4, 5)
        return (0, 1, 2, 3, 4, 5)

    @property
    def group_width(self) -> int:
        return len(self.field_indices)


def max_bits_per_field(group_width: int) -> int:
    return 21 if group_width == 3 else 64 // group_width


@dataclass(frozen=True)
class Segment:
    start: int
    end: int
    bits: int
    minima: Tuple[int, ...]

    @property
    def count(self) -> int:
        return self.end - self.start


def segment_bounds(n: int, segment_size: int) -> np.ndarray:
    if segment_size < 1:
        raise ValidationError("segment_size must be >= 1")
    starts = list(range(0, n, segment_size)) + [n]
    if n == 0:
        starts = [0, 0]
    return np.array(starts, np.int64)
