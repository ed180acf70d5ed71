"""A100 MIG profile pick — drop-in for the reference mig.py:1-45.

The rule (smallest profile whose ceiling covers the predicted memory, upper
bounds inclusive, 1 GB = 1024 MB, <=0 or >40960 -> None, NaN/Inf ->
NonFinite) lives once in the native library as a __host__ __device__
function: `mig_profile` calls its host instance through the C ABI, and the
batched prediction path evaluates the same function on the device inside the
head kernel (dippm_head_forward), so scalar and batched picks cannot diverge.
"""

from __future__ import annotations

import ctypes
import enum

from . import _lib


class MigProfile(enum.Enum):
    """A100 partition sizes, ordered by memory ceiling (mig.py:16-29)."""

    MIG_1G_5GB = ("1g.5gb", 5 * 1024)
    MIG_2G_10GB = ("2g.10gb", 10 * 1024)
    MIG_3G_20GB = ("3g.20gb", 20 * 1024)
    MIG_7G_40GB = ("7g.40gb", 40 * 1024)

    def __init__(self, label: str, max_memory_mb: int):
        self.label = label
        self.max_memory_mb = max_memory_mb

    def __str__(self) -> str:
        return self.label


_BY_CODE = list(MigProfile)


def profile_from_code(code: int) -> MigProfile | None:
    """Map a kernel MIG code (0..3, -1 = None) to the enum."""
    return None if code < 0 else _BY_CODE[code]


def mig_profile(alpha_mb: float) -> MigProfile | None:
    """Smallest profile whose memory ceiling covers alpha_mb (mig.py:32-45).

    Returns None for alpha_mb <= 0 or above 40960 MB; raises NonFinite for
    NaN or infinite input.
    """
    code = ctypes.c_int32(-1)
    _lib.check(_lib.load().dippm_mig_code(float(alpha_mb), ctypes.byref(code)), "mig_profile")
    return profile_from_code(code.value)
