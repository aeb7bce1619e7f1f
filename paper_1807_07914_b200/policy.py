"""Truncation rule applied after every two-site SVD.

Same dataclass, defaults, validation messages and keep rule as the reference
``TruncationPolicy`` (``R:src/mpsqvm/mps.py:24-49``). On the device the rule is
evaluated by ``finalize_kernel`` (``csrc/bmps_update.cuh``); ``keep_count`` here
is the host-side mirror for callers that inspect spectra themselves.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._native import BmpsPolicy


@dataclass(frozen=True)
class TruncationPolicy:
    """Discard sigma below ``cutoff * sigma_max`` (relative) or ``cutoff``
    (absolute), then cap at ``max_bond``; keep at least one value."""

    cutoff: float = 1e-4
    max_bond: int | None = None
    relative: bool = True

    def __post_init__(self) -> None:
        if self.cutoff < 0:
            raise ValueError("cutoff must be >= 0")
        if self.max_bond is not None and self.max_bond < 1:
            raise ValueError("max_bond must be >= 1")

    def keep_count(self, singular_values: np.ndarray) -> int:
        s = np.asarray(singular_values)
        if self.cutoff > 0:
            thr = self.cutoff * (s[0] if self.relative else 1.0)
            keep = int(np.count_nonzero(s >= thr))
        else:
            keep = len(s)
        keep = max(keep, 1)
        return keep if self.max_bond is None else min(keep, self.max_bond)

    def as_c(self) -> BmpsPolicy:
        return BmpsPolicy(float(self.cutoff), int(self.max_bond or 0), 1 if self.relative else 0)
