"""bf16 <-> fp32 helpers on numpy uint16 storage (round-to-nearest-even, as __float2bfloat16_rn)."""
import numpy as np


def to_bf16(a) -> np.ndarray:
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    r = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + r) >> 16).astype(np.uint16)


def from_bf16(b) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def round_bf16(a) -> np.ndarray:
    return from_bf16(to_bf16(a))
