"""Race arbitration policy of the barrier-phase model (parallel/engine.py:47-94).

The reference executes the paper's kernels as Python phase programs and
resolves same-cell writes with an ``Arbitration``; on the GPU the only racy
write that changes the LexBFS order is the election of ``current`` among the
members of the max-label set (parallel/lexbfs.py:211-225), and the kernel
implements that election directly from the policy below (``tie_rule``).
"""

from __future__ import annotations

from dataclasses import dataclass

from .. import _native

NULL = -1
_MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """splitmix64 finaliser (_bitops.py:43-49)."""
    x = (x + 0x9E3779B97F4A7C15) & _MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK64
    return x ^ (x >> 31)


def mix64(*values: int) -> int:
    """Order-sensitive fold of integers into 64 bits (_bitops.py:51-57)."""
    h = 0
    for v in values:
        h = splitmix64(h ^ (int(v) & _MASK64))
    return h


def label_hash(text: str) -> int:
    import zlib

    return zlib.crc32(text.encode("ascii"))


@dataclass(frozen=True)
class Arbitration:
    """Policy resolving racy same-cell writes within a phase."""

    mode: str  # "seeded" or "fixed"
    seed: int | None = None
    direction: str = "ascending"

    @classmethod
    def seeded(cls, seed: int) -> "Arbitration":
        return cls("seeded", seed=int(seed))

    @classmethod
    def fixed_priority(cls, direction: str = "ascending") -> "Arbitration":
        if direction not in ("ascending", "descending"):
            raise ValueError(f"direction must be ascending or descending, got {direction!r}")
        return cls("fixed", direction=direction)

    def choose(self, table: str, index: int, epoch: int, writers) -> int:
        """Winning task id for one contested cell (engine.py:65-71)."""
        if self.mode == "fixed":
            return min(writers) if self.direction == "ascending" else max(writers)
        prefix = mix64(self.seed, epoch, mix64(label_hash(table), index))
        return max(writers, key=lambda w: (splitmix64(prefix ^ w), w))

    @property
    def tie_rule(self) -> int:
        """The kernel's election rule for this policy (include/chordal_b200.h)."""
        if self.mode == "fixed":
            return _native.TIE_ASCENDING if self.direction == "ascending" else _native.TIE_DESCENDING
        if self.mode == "seeded":
            return _native.TIE_SEEDED_ARB
        raise ValueError(f"unknown arbitration mode {self.mode!r}")
