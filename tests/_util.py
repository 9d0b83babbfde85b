"""Shared helpers for the test-suite (fixtures, bf16 round-trips, error metric)."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def golden(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def bf16f(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def to_bf16_bits(a) -> np.ndarray:
    f = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    rounded = f + np.uint32(0x7FFF) + ((f >> np.uint32(16)) & np.uint32(1))
    return (rounded >> np.uint32(16)).astype(np.uint16)


def rel_err(got, ref) -> float:
    """max|got-ref| / max|ref| -- the reference's error convention (model.py:289-297)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))


def torch_bf16(bits: np.ndarray, device="cuda"):
    import torch

    t = torch.from_numpy(bits.astype(np.int16).view(np.int16).copy())
    return t.view(torch.bfloat16).to(device)


def fp16_round(a: np.ndarray) -> np.ndarray:
    return np.asarray(a, np.float64).astype(np.float16).astype(np.float64)


def unpack_rows(rows: np.ndarray, bits: int, cols: int) -> np.ndarray:
    """Codes of LSB-first packed arena rows (uint8 [n, row_bytes]) -> uint8 [n, cols]."""
    b = np.unpackbits(rows, axis=1, bitorder="little")[:, :cols * bits].reshape(len(rows), cols, bits)
    return (b.astype(np.uint8) << np.arange(bits, dtype=np.uint8)).sum(axis=2, dtype=np.uint8)
