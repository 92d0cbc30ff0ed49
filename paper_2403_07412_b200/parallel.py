"""Worker-count API of the reference (vg/parallel.py:15-43), kept for drop-in
compatibility.  On the B200 path the CUDA grid replaces the thread pool and
results are launch-configuration independent by construction (fixed
4096-entry reduction chunks, per-entry arithmetic that never mixes entries),
so the setting has no effect on any result.
"""

from __future__ import annotations

_num_threads = 1


def set_num_threads(n: int) -> None:
    global _num_threads
    if n < 1:
        raise ValueError(f"thread count must be >= 1, got {n}")
    _num_threads = int(n)


def get_num_threads() -> int:
    return _num_threads


def chunk_ranges(start: int, stop: int, chunk: int) -> list[tuple[int, int]]:
    """Half-open ranges covering [start, stop) in steps of `chunk` (vg/parallel.py:30-34)."""
    if chunk < 1:
        raise ValueError("chunk must be >= 1")
    return [(s, min(s + chunk, stop)) for s in range(start, stop, chunk)]
