"""Byte-size literals for ``memory_limit`` and the CLI size flags.

The accepted language is the reference's (cli.py:33-68): a
non-negative number, optionally fractional, followed by an optional unit -
``B``, decimal ``KB``/``MB``/``GB`` (powers of ten) or binary
``KiB``/``MiB``/``GiB`` (powers of two), case-insensitive - that denotes a
whole number of bytes; a unit-less literal must be a plain integer.  Parsing
here is a single regular expression with exact decimal arithmetic.
"""

from __future__ import annotations

import re
from decimal import Decimal, InvalidOperation

_UNITS = {"": 1, "b": 1, "kb": 10**3, "mb": 10**6, "gb": 10**9,
          "kib": 1 << 10, "mib": 1 << 20, "gib": 1 << 30}
_LITERAL = re.compile(r"^\s*(?P<num>\d+(?:\.\d*)?|\.\d+)\s*(?P<unit>[kmg]i?b|b)?\s*$",
                      re.IGNORECASE)
# rendering order: decimal units first, then binary, largest first
_RENDER = (("GB", 10**9), ("MB", 10**6), ("KB", 10**3),
           ("GiB", 1 << 30), ("MiB", 1 << 20), ("KiB", 1 << 10))


def parse_size(text) -> int:
    """'1GB' -> 10**9, '64MiB' -> 64 * 2**20, '512' -> 512 (bytes)."""
    if isinstance(text, bool):
        raise ValueError(f"not a size literal: {text!r}")
    if isinstance(text, int):
        if text < 0:
            raise ValueError("a size cannot be negative")
        return text
    match = _LITERAL.match(str(text))
    if match is None:
        raise ValueError(f"not a size literal: {text!r}")
    unit = (match.group("unit") or "").lower()
    number = match.group("num")
    if not unit and not number.isdigit():
        raise ValueError(f"a size without a unit must be an integer byte count: {text!r}")
    try:
        value = Decimal(number) * _UNITS[unit]
    except InvalidOperation as exc:                 # pragma: no cover - regex guards it
        raise ValueError(f"not a size literal: {text!r}") from exc
    if value != value.to_integral_value():
        raise ValueError(f"{text!r} is a fraction of a byte")
    return int(value)


def format_size(nbytes: int) -> str:
    """Shortest exact literal: the largest unit that divides the count,
    decimal before binary; plain bytes otherwise."""
    if nbytes < 0:
        raise ValueError("a size cannot be negative")
    for unit, scale in _RENDER:
        q, r = divmod(nbytes, scale)
        if nbytes and r == 0:
            return f"{q}{unit}"
    return f"{nbytes}B"


def as_limit(memory_limit) -> int:
    """None -> 0 (no limit), otherwise the parsed byte count (> 0)."""
    if memory_limit is None:
        return 0
    nbytes = parse_size(memory_limit)
    if nbytes <= 0:
        raise ValueError("memory_limit must be a positive byte count")
    return nbytes
