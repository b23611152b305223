"""Score policies (scoring.py:27-53 of the reference): host-side enums and the
caller-advanced epoch.  The per-key score arithmetic itself runs in the
kernels (csrc/hkv_common.cuh: insert_score / hit_score)."""

from __future__ import annotations

import enum

MAX_SCORE = 0xFFFFFFFFFFFFFFFF
_LOW32 = 0xFFFFFFFF


class PolicyId(enum.Enum):
    kLru = "kLru"
    kLfu = "kLfu"
    kEpochLru = "kEpochLru"
    kEpochLfu = "kEpochLfu"
    kCustomized = "kCustomized"


ALL_POLICIES = tuple(PolicyId)


class EpochState:
    """Caller-advanced epoch; may only move forward (scoring.py:38-53)."""

    __slots__ = ("current_epoch",)

    def __init__(self, current_epoch: int = 0):
        if current_epoch < 0 or current_epoch > _LOW32:
            raise ValueError("epoch must fit in 32 bits")
        self.current_epoch = current_epoch

    def advance_to(self, epoch: int) -> None:
        if epoch < self.current_epoch:
            raise ValueError("epoch may not decrease")
        if epoch > _LOW32:
            raise ValueError("epoch must fit in 32 bits")
        self.current_epoch = epoch
