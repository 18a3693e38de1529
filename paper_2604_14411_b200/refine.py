"""Refinement payload types (refine.py:44-67 of the reference).

The rounds themselves run on the GPU inside ``dhgp_partition``; ``MoveSet``
and ``PrefixSelection`` carry each round's sequence and selection to the
observer with the reference's field names and dtypes.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

__all__ = ["MoveSet", "PrefixSelection"]


@dataclass(frozen=True)
class MoveSet:
    """Gain-sorted move sequence: descending ``gain_iso``, ties toward the
    smaller node id; ``gain_seq`` assumes all earlier moves applied."""

    node: np.ndarray
    from_part: np.ndarray
    to_part: np.ndarray
    gain_iso: np.ndarray
    gain_seq: np.ndarray | None = None

    def __len__(self) -> int:
        return len(self.node)


class PrefixSelection(NamedTuple):
    k: int
    total_gain: float
    active: np.ndarray  # violation count after each prefix, len(moves) + 1
