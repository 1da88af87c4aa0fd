"""Packed GF(2) vectors in the reference's wire layout.

A vector of L bits is ``ceil(L/64)`` little-endian uint64 words with bit ``i``
at ``(words[i >> 6] >> (i & 63)) & 1`` — exactly ``qldpc::Gf2Vector::words()``
(reference: proj/include/qldpc/gf2.hpp:13-67), which is what crosses the C-ABI.
"""
from __future__ import annotations

import numpy as np


def num_words(bits: int) -> int:
    return (int(bits) + 63) // 64


def pack_bits(bits: np.ndarray) -> np.ndarray:
    """(..., L) array of 0/1 -> (..., ceil(L/64)) uint64 words."""
    bits = np.asarray(bits, dtype=np.uint8)
    length = bits.shape[-1]
    pad = num_words(length) * 64 - length
    if pad:
        bits = np.concatenate(
            [bits, np.zeros(bits.shape[:-1] + (pad,), dtype=np.uint8)], axis=-1)
    packed = np.packbits(bits, axis=-1, bitorder="little")
    return np.ascontiguousarray(packed).view("<u8")


def unpack_bits(words: np.ndarray, length: int) -> np.ndarray:
    """(..., W) uint64 words -> (..., length) uint8 bits."""
    words = np.ascontiguousarray(np.asarray(words, dtype="<u8"))
    as_bytes = words.view(np.uint8)
    bits = np.unpackbits(as_bytes, axis=-1, bitorder="little")
    return bits[..., :length]


def concat_bits(a_words: np.ndarray, a_len: int, b_words: np.ndarray, b_len: int) -> np.ndarray:
    """Gf2Vector::concat (gf2.hpp:56): a followed by b, re-packed."""
    a = unpack_bits(a_words, a_len)
    b = unpack_bits(b_words, b_len)
    return pack_bits(np.concatenate([a, b], axis=-1))


def to_hex(words: np.ndarray, length: int) -> str:
    """Gf2Vector::to_hex (gf2.hpp:61): digit j encodes bits [4j, 4j+4), LSB first."""
    bits = unpack_bits(words, length)
    digits = []
    for j in range((length + 3) // 4):
        nib = 0
        for b in range(4):
            idx = 4 * j + b
            if idx < length and bits[idx]:
                nib |= 1 << b
        digits.append("0123456789abcdef"[nib])
    return "".join(digits)
