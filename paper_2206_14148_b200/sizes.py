"""Size literals with the reference's semantics (cli.py:33-68):
decimal KB/MB/GB are powers of ten, KiB/MiB/GiB powers of two, bare digits
are bytes.  ``memory_limit`` accepts these literals everywhere."""

from __future__ import annotations

_DECIMAL = {"B": 1, "KB": 10**3, "MB": 10**6, "GB": 10**9}
_BINARY = {"KIB": 2**10, "MIB": 2**20, "GIB": 2**30}
_ALL = sorted({**_DECIMAL, **_BINARY}.items(), key=lambda kv: -len(kv[0]))


def parse_size(text) -> int:
    """'1GB' -> 10**9, '64MiB' -> 64 * 2**20, bare digits -> bytes."""
    if isinstance(text, bool):
        raise ValueError(f"malformed size literal {text!r}")
    if isinstance(text, int):
        if text < 0:
            raise ValueError("sizes are non-negative")
        return text
    s = str(text).strip()
    upper = s.upper()
    for suffix, mult in _ALL:
        if upper.endswith(suffix):
            number = s[: len(s) - len(suffix)].strip()
            if not number:
                raise ValueError(f"missing number in size literal {text!r}")
            result = float(number) * mult
            if result != int(result) or result < 0:
                raise ValueError(f"size literal {text!r} is not a whole byte count")
            return int(result)
    if not s.isdigit():
        raise ValueError(f"malformed size literal {text!r}")
    return int(s)


def format_size(nbytes: int) -> str:
    """Largest suffix that divides exactly, preferring decimal."""
    if nbytes < 0:
        raise ValueError("sizes are non-negative")
    for suffix, mult in (("GB", 10**9), ("MB", 10**6), ("KB", 10**3)):
        if nbytes and nbytes % mult == 0:
            return f"{nbytes // mult}{suffix}"
    for suffix, mult in (("GiB", 2**30), ("MiB", 2**20), ("KiB", 2**10)):
        if nbytes and nbytes % mult == 0:
            return f"{nbytes // mult}{suffix}"
    return f"{nbytes}B"


def as_limit(memory_limit) -> int:
    """None -> 0 (unlimited), else parsed bytes (must be positive)."""
    if memory_limit is None:
        return 0
    v = parse_size(memory_limit)
    if v <= 0:
        raise ValueError("memory_limit must be a positive byte count")
    return v
