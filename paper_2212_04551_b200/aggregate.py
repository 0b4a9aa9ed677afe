"""Host side of leaf aggregation: pattern counters and the record stream.

Mirrors the public helpers of ``warpmine.aggregate`` (reference
``pkg/src/warpmine/aggregate.py``).  The per-leaf work itself
(``count_valid`` / ``aggregate_pattern`` / ``aggregate_store``) runs on the
device (``csrc/wm_motif.cu``, ``csrc/wm_clique.cu``); what stays on the host is

* ``PatternCounter`` / ``reduce_counts`` (``aggregate.py:18-55``) for callers
  that sum per-part histograms themselves,
* ``format_record`` (``aggregate.py:64-66``), the CLI rendering of a record,
* ``StoreBuffer`` (``aggregate.py:69-147``), the bounded producer/consumer
  channel between the enumeration and the user's sink.  On B200 the producer
  is the listing drain loop of ``wm_run_listing``: device warps block on the
  device ring while the host side of the chain (this buffer) is full, so
  back-pressure reaches the GPU.
"""

from __future__ import annotations

import collections
import threading
from typing import Callable, Iterable, Optional

from .errors import StoreShutdownError


class PatternCounter:
    """Dense per-pattern counter addressed by dictionary id
    (reference ``aggregate.py:18-36``)."""

    __slots__ = ("counts",)

    def __init__(self, pattern_count: int):
        if pattern_count < 1:
            raise ValueError("pattern_count must be positive")
        self.counts = [0] * pattern_count

    def add(self, pattern_id: int, amount: int = 1) -> None:
        self.counts[pattern_id] += amount

    def total(self) -> int:
        return sum(self.counts)

    def __len__(self):
        return len(self.counts)


def reduce_counts(parts: Iterable) -> list:
    """Elementwise sum of equally long histograms or PatternCounters
    (reference ``aggregate.py:39-55``); ``[]`` for no parts."""
    total = None
    for part in parts:
        row = list(part.counts if isinstance(part, PatternCounter) else part)
        if total is None:
            total = row
            continue
        if len(row) != len(total):
            raise ValueError("counter length mismatch")
        total = [a + b for a, b in zip(total, row)]
    return total if total is not None else []


def adjacency_mask(tr, length: int, adj_set) -> int:
    """Bit j set iff ``tr[j]`` is in ``adj_set`` (reference ``aggregate.py:160-166``)."""
    return sum(1 << j for j in range(length) if tr[j] in adj_set)


def format_record(vertices, bits: int) -> str:
    """One emitted subgraph: ascending vertex ids, then the bitmap in hex
    (reference ``aggregate.py:64-66``)."""
    return " ".join(map(str, sorted(vertices))) + " 0x%x" % bits


_END = object()


class StoreBuffer:
    """Bounded channel for emitted records (reference ``aggregate.py:69-147``).

    ``put`` blocks while ``capacity`` records are waiting, so production runs
    no faster than the consumer drains.  If the consumer's sink raises, the
    buffer is marked failed and every later ``put`` raises
    ``StoreShutdownError`` instead of blocking forever.
    """

    def __init__(self, capacity: int = 1024):
        if capacity < 1:
            raise ValueError("capacity must be positive")
        self.capacity = capacity
        self._items: collections.deque = collections.deque()
        self._cv = threading.Condition()
        self._failed = False
        self._closed = False
        self._thread: Optional[threading.Thread] = None
        self.consumed = 0

    def put(self, record) -> None:
        with self._cv:
            if self._closed:
                raise StoreShutdownError("store buffer already closed")
            while len(self._items) >= self.capacity and not self._failed:
                self._cv.wait(0.05)
            if self._failed:
                raise StoreShutdownError("store consumer terminated")
            self._items.append(record)
            self._cv.notify_all()

    def close(self) -> None:
        """End of stream; idempotent."""
        with self._cv:
            if self._closed:
                return
            self._closed = True
            self._items.append(_END)  # the end marker may exceed capacity by one
            self._cv.notify_all()

    def drain(self, sink: Callable) -> int:
        """Apply ``sink`` to each record until the stream is closed; returns
        the number consumed.  A raising sink marks the buffer failed and the
        exception propagates."""
        done = 0
        while True:
            with self._cv:
                while not self._items:
                    self._cv.wait()
                item = self._items.popleft()
                self._cv.notify_all()
            if item is _END:
                return done
            try:
                sink(item)
            except BaseException:
                with self._cv:
                    self._failed = True
                    self._cv.notify_all()
                raise
            done += 1
            self.consumed = done

    def start_consumer(self, sink: Callable) -> threading.Thread:
        if self._thread is not None:
            raise RuntimeError("consumer already started")

        def consume():
            try:
                self.drain(sink)
            except BaseException:
                pass  # recorded in self._failed; producers see StoreShutdownError

        self._thread = threading.Thread(target=consume, name="store-consumer", daemon=True)
        self._thread.start()
        return self._thread

    def join(self, timeout: float = 30.0) -> None:
        """Close the stream and wait for the consumer."""
        self.close()
        if self._thread is not None:
            self._thread.join(timeout=timeout)
            if self._thread.is_alive():
                raise StoreShutdownError("store consumer failed to drain")

    @property
    def failed(self) -> bool:
        return self._failed
