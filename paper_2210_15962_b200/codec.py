"""Half-sequence packing and the hex code of published sequences.

Bit contract shared with the device (and with skewsaw.codec, codec.py:34-90):
a half sequence of D spins is the D-bit integer whose most significant bit is
spin 0, with -1 -> 1 and +1 -> 0; the hex text is that integer zero-padded to
ceil(D/4) nibbles with a ``0x`` prefix.  The device's packed ``words`` are the
same integer split into little-endian uint64 words.
"""

from __future__ import annotations

import numpy as np

from .core import as_spins, half_dim

__all__ = ["DecodeError", "encode", "decode", "pack_half", "unpack_half", "parse_record_line"]


class DecodeError(ValueError):
    """Hex text that cannot be the half sequence of the declared length."""


def pack_half(half) -> int:
    spins = as_spins(half)
    bits = "".join("1" if v < 0 else "0" for v in spins.tolist())
    return int(bits, 2)


def unpack_half(value: int, d: int) -> np.ndarray:
    if value < 0 or value.bit_length() > d:
        raise ValueError(f"value does not fit in {d} bits")
    bits = format(value, f"0{d}b") if d > 0 else ""
    return np.fromiter((-1 if b == "1" else 1 for b in bits), dtype=np.int64, count=d)


def encode(half) -> str:
    spins = as_spins(half)
    width = -(-spins.size // 4)
    return "0x" + format(pack_half(spins), f"0{width}X")


def decode(text: str, length: int) -> np.ndarray:
    if length < 1 or length % 2 == 0:
        raise DecodeError(f"declared length must be odd, got {length}")
    d = half_dim(length)
    body = text.strip()
    if body[:2].lower() == "0x":
        body = body[2:]
    if not body:
        raise DecodeError("empty hex string")
    try:
        value = int(body, 16)
    except ValueError:
        raise DecodeError(f"not a hexadecimal string: {text!r}") from None
    if value.bit_length() > d:
        raise DecodeError(f"hex value needs {value.bit_length()} bits but length {length} allows only {d}")
    return unpack_half(value, d)


def parse_record_line(line: str):
    """``L 0xHEX [E [F]]`` -> (L, hex, E or None, F or None)."""
    parts = line.split()
    if not 2 <= len(parts) <= 4:
        raise ValueError("expected `L 0xHEX [E [F]]`")
    conv = [int, str, int, float]
    names = ["length", "hex", "energy", "merit factor"]
    out = []
    for i, tok in enumerate(parts):
        try:
            out.append(conv[i](tok))
        except ValueError:
            raise ValueError(f"bad {names[i]} field {tok!r}") from None
    out += [None] * (4 - len(out))
    return tuple(out)
