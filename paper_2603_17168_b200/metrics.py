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


_FIELDS = [f.name for f in fields(TxnCounters)]


class DeviceTxnCounters(TxnCounters):
    """`CacheTable.counters`: a live view of the table's device counters
    (hkv_counters / hkv_reset_counters), so the reference callers' pattern
    `table.counters.reset(); ...; table.counters.digest_line_loads`
    (bench.py:198-205, 556-558; service.py:282-289) reads what the kernels
    counted since the reset.  Assigning a field or merge() adds a host-side
    offset, like mutating the reference's dataclass."""

    def __init__(self, table):  # noqa: D401 - not the dataclass __init__
        object.__setattr__(self, "_table", table)
        object.__setattr__(self, "_offset", dict.fromkeys(_FIELDS, 0))

    def _device(self) -> dict:
        return self._table._device_counters()

    def __getattribute__(self, name):
        if name in _FIELDS:
            return object.__getattribute__(self, "_device")()[name] + object.__getattribute__(self, "_offset")[name]
        return object.__getattribute__(self, name)

    def __setattr__(self, name, value):
        if name in _FIELDS:
            self._offset[name] = int(value) - self._device()[name]
            return
        object.__setattr__(self, name, value)

    def as_dict(self) -> dict:
        d = self._device()
        return {k: d[k] + self._offset[k] for k in _FIELDS}

    def snapshot(self) -> TxnCounters:
        return TxnCounters(**self.as_dict())

    def reset(self) -> None:
        self._table.reset_counters()
        for k in _FIELDS:
            self._offset[k] = 0

    def merge(self, other: TxnCounters) -> None:
        for k in _FIELDS:
            self._offset[k] += getattr(other, k)

    @property
    def value_copies(self) -> int:
        d = self.as_dict()
        return d["value_copies_fast"] + d["value_copies_overflow"]

    def __repr__(self) -> str:
        return "DeviceTxnCounters(" + ", ".join(f"{k}={v}" for k, v in self.as_dict().items()) + ")"

    def __eq__(self, other) -> bool:
        if isinstance(other, TxnCounters):
            return self.as_dict() == {k: getattr(other, k) for k in _FIELDS}
        return NotImplemented

    __hash__ = None
