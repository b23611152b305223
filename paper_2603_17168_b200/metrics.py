"""TxnCounters (metrics.py:14-39 of the reference): structural cost counters
maintained on the device by every kernel (one block-reduced atomicAdd per
counter per block) and read back on demand."""

from __future__ import annotations

from dataclasses import dataclass, fields


@dataclass
class TxnCounters:
    digest_line_loads: int = 0
    full_key_compares: int = 0
    score_scans: int = 0
    slot_lock_retries: int = 0
    value_copies_fast: int = 0
    value_copies_overflow: int = 0

    def merge(self, other: "TxnCounters") -> None:
        for f in fields(self):
            setattr(self, f.name, getattr(self, f.name) + getattr(other, f.name))

    def snapshot(self) -> "TxnCounters":
        return TxnCounters(**self.as_dict())

    def reset(self) -> None:
        for f in fields(self):
            setattr(self, f.name, 0)

    def as_dict(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}

    @property
    def value_copies(self) -> int:
        return self.value_copies_fast + self.value_copies_overflow
