"""paper_2603_17168_b200 — B200-native cache-semantic hash table (HierarchicalKV).

Drop-in for the reference `cachekv` table API (/root/reference/pkg/src/cachekv/
__init__.py:9-52): CacheTable, TableConfig, Mode, Outcome, PolicyId, ...
backed by sm_100a kernels through the C-ABI in include/hkv_b200.h.
"""

from .gate import ROLE_OF_OPERATION, Role, RoleGate, RoleGuard
from .metrics import TxnCounters
from .scoring import ALL_POLICIES, MAX_SCORE, EpochState, PolicyId
from .table import (
    BUCKET_SLOTS,
    EMPTY_KEY,
    LOCKED_KEY,
    CacheTable,
    ConsistencyError,
    LookupResult,
    Mode,
    Outcome,
    TableConfig,
    Tier,
    UpsertResult,
    ValueHandle,
)

__all__ = [
    "ALL_POLICIES", "BUCKET_SLOTS", "CacheTable", "ConsistencyError", "EMPTY_KEY", "EpochState", "LOCKED_KEY",
    "LookupResult", "MAX_SCORE", "Mode", "Outcome", "PolicyId", "ROLE_OF_OPERATION", "Role", "RoleGate", "RoleGuard",
    "TableConfig", "Tier", "TxnCounters", "UpsertResult", "ValueHandle",
]

__version__ = "0.1.0"
