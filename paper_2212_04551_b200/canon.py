"""Induced-edge bitmaps, canonical forms and the pattern dictionary (host side).

Encoding (reference ``pkg/src/warpmine/canon.py:1-20``, ``:50-90``): for a
traversal ``v_0..v_{k-1}`` the edge ``(v_i, v_j)``, ``j < i``, ``i >= 2``, sits
at bit ``i(i-1)/2 - 1 + j``; the ``(v_0, v_1)`` edge is implicit.  Appending
position ``p`` with adjacency mask ``m`` ORs ``m << (p(p-1)/2 - 1)``.

The dictionary maps every reachable ``k``-vertex bitmap to a dense pattern id
(ids ascend with the class-minimum bitmap, so the complete graph is the last
id) and unreachable bitmaps to ``SENTINEL``.  The device kernels index this
exact u32 table (uploaded per run), so it must be byte-identical to the
reference's ``build_dictionary`` output — ``tests/test_canon.py`` pins that
against SHA-256 digests generated from the reference.

Construction here is an orbit sweep like the reference's
(``canon.py:315-343``): walk valid bitmaps ascending, and the first unlabelled
one is its class minimum; label its whole orbit at once.  The orbit is computed
from a per-permutation edge-slot map held as a ``(k!, nbits+1)`` uint64 mask
matrix.
"""

from __future__ import annotations

import itertools
import struct
from dataclasses import dataclass
from functools import lru_cache
from typing import Sequence

import numpy as np

from .errors import DictionaryFormatError

SENTINEL = 0xFFFFFFFF
_MAGIC = b"DMCD"
_VERSION = 1

K_MAX_DEFAULT = 7
K_MAX_LARGE = 8


def group_offset(i: int) -> int:
    """Bit offset of vertex group ``i >= 2`` (reference ``canon.py:50-52``)."""
    return i * (i - 1) // 2 - 1


def stored_bits(k: int) -> int:
    """Stored bits of a k-vertex bitmap (reference ``canon.py:55-57``)."""
    return k * (k - 1) // 2 - 1


@dataclass(frozen=True)
class EdgeBitmap:
    bits: int
    k: int

    def __post_init__(self):
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if self.k >= 2 and self.bits >> stored_bits(self.k):
            raise ValueError("bits 0x%x exceed %d stored bits for k=%d"
                             % (self.bits, stored_bits(self.k), self.k))
        if self.k < 2 and self.bits:
            raise ValueError("k<2 bitmaps store no bits")


def extend_bits(bits: int, k: int, adjacency_bits: int) -> int:
    """Bitmap of ``k+1`` vertices from a ``k``-vertex bitmap and the new
    vertex's k-bit adjacency mask (reference ``canon.py:76-90``)."""
    if adjacency_bits == 0:
        raise ValueError("appended vertex must neighbor the traversal (mask is 0)")
    if adjacency_bits >> k:
        raise ValueError("adjacency mask 0x%x wider than k=%d" % (adjacency_bits, k))
    if k == 1:
        return 0
    return bits | (adjacency_bits << group_offset(k))


def encode_extension(b: EdgeBitmap, adjacency_bits: int) -> EdgeBitmap:
    return EdgeBitmap(extend_bits(b.bits, b.k, adjacency_bits), b.k + 1)


def bitmap_is_valid(bits: int, k: int) -> bool:
    """Every vertex group ``i >= 2`` non-empty (reference ``canon.py:107-112``)."""
    return all((bits >> group_offset(i)) & ((1 << i) - 1) for i in range(2, k))


# ---------------------------------------------------------------------------
# relabelling


@lru_cache(maxsize=None)
def _slot_maps(k: int):
    """``masks[p, s]`` = one-hot u64 of the slot that source slot ``s`` moves
    to under permutation ``p``.  Slot ``nbits`` is the implicit (1,0) edge."""
    nbits = stored_bits(k)
    hi = np.array([i for i in range(1, k) for j in range(i)], dtype=np.int64)
    lo = np.array([j for i in range(1, k) for j in range(i)], dtype=np.int64)
    src_slot = np.where(hi == 1, nbits, hi * (hi - 1) // 2 - 1 + lo)
    perms = np.array(list(itertools.permutations(range(k))), dtype=np.int64)
    a, b = perms[:, hi], perms[:, lo]
    ph, pl = np.maximum(a, b), np.minimum(a, b)
    dst_slot = np.where(ph == 1, nbits, ph * (ph - 1) // 2 - 1 + pl)
    masks = np.zeros((len(perms), nbits + 1), dtype=np.uint64)
    masks[:, src_slot] = np.left_shift(np.uint64(1), dst_slot.astype(np.uint64))
    groups = [(np.uint64(group_offset(i)), np.uint64((1 << i) - 1)) for i in range(2, k)]
    return nbits, masks, groups


def _orbit(bits: int, k: int):
    """(stored images, valid flags) of ``bits`` under all k! relabelings."""
    nbits, masks, groups = _slot_maps(k)
    full = bits | (1 << nbits)
    cols = [s for s in range(nbits + 1) if (full >> s) & 1]
    img = np.bitwise_or.reduce(masks[:, cols], axis=1)
    ok = ((img >> np.uint64(nbits)) & np.uint64(1)) == np.uint64(1)
    for sh, w in groups:
        ok &= ((img >> sh) & w) != np.uint64(0)
    return img & np.uint64((1 << nbits) - 1), ok


def canonical_bits(bits: int, k: int) -> int:
    """Minimum valid relabelled bitmap (reference ``canon.py:170-178``)."""
    if k < 3:
        raise ValueError("canonical form needs k >= 3, got k=%d" % k)
    if not bitmap_is_valid(bits, k):
        raise ValueError("bitmap 0x%x encodes a disconnected traversal" % bits)
    img, ok = _orbit(bits, k)
    return int(img[ok].min())


def canonical_form(b: EdgeBitmap) -> EdgeBitmap:
    return EdgeBitmap(canonical_bits(b.bits, b.k), b.k)


def is_canonical_candidate(tr: Sequence[int], u: int, g) -> bool:
    """Canonical-candidate rule (reference ``canon.py:190-210``): ``u >
    tr[0]`` and, with ``f`` the first position adjacent to ``u``, ``u >
    tr[j]`` for all ``j > f``."""
    if u <= tr[0]:
        return False
    first = next((j for j, v in enumerate(tr) if g.has_edge(u, v)), -1)
    if first < 0:
        return False
    return all(u > tr[j] for j in range(first + 1, len(tr)))


# ---------------------------------------------------------------------------
# dictionary


class CanonicalDictionary:
    """Bitmap -> pattern id table (reference ``canon.py:217-296``)."""

    __slots__ = ("k", "table", "pattern_count", "canonical_bitmaps", "_fast", "__weakref__")

    def __init__(self, k: int, table: np.ndarray, canonical_bitmaps: list):
        self.k = k
        self.table = np.ascontiguousarray(table, dtype=np.uint32)
        self.pattern_count = len(canonical_bitmaps)
        self.canonical_bitmaps = list(canonical_bitmaps)
        self._fast = None

    def lookup(self, b: EdgeBitmap) -> int:
        if b.k != self.k:
            raise ValueError("bitmap is for k=%d, dictionary for k=%d" % (b.k, self.k))
        return int(self.table[b.bits])

    def fast_table(self):
        if self._fast is None:
            self._fast = self.table.tolist() if self.k <= K_MAX_DEFAULT else self.table
        return self._fast

    def to_bytes(self) -> bytes:
        """DMCD v1 bytes (reference ``canon.py:249-257``): magic, u8 version,
        u8 k, u64 table length, u32 table, u32 pattern count, u64 bitmaps."""
        return b"".join([
            _MAGIC, bytes([_VERSION, self.k]), struct.pack("<Q", len(self.table)),
            self.table.astype("<u4").tobytes(),
            struct.pack("<I", self.pattern_count),
            np.asarray(self.canonical_bitmaps, dtype="<u8").tobytes()])

    def save(self, path) -> None:
        with open(path, "wb") as fh:
            fh.write(self.to_bytes())

    @classmethod
    def from_bytes(cls, blob: bytes) -> "CanonicalDictionary":
        """Validate and parse DMCD bytes (reference ``canon.py:259-293``)."""
        if len(blob) < 14:
            raise DictionaryFormatError("file too short (%d bytes)" % len(blob))
        if blob[:4] != _MAGIC:
            raise DictionaryFormatError("bad magic %r" % blob[:4])
        version, k = blob[4], blob[5]
        if version != _VERSION:
            raise DictionaryFormatError("unsupported version %d" % version)
        if not 3 <= k <= K_MAX_LARGE:
            raise DictionaryFormatError("k=%d outside supported range 3..%d" % (k, K_MAX_LARGE))
        (tlen,) = struct.unpack_from("<Q", blob, 6)
        if tlen != 1 << stored_bits(k):
            raise DictionaryFormatError("table length %d inconsistent with k=%d (expected %d)"
                                        % (tlen, k, 1 << stored_bits(k)))
        end_table = 14 + 4 * tlen
        if len(blob) < end_table + 4:
            raise DictionaryFormatError("truncated table")
        table = np.frombuffer(blob, "<u4", tlen, 14).copy()
        (pc,) = struct.unpack_from("<I", blob, end_table)
        if len(blob) != end_table + 4 + 8 * pc:
            raise DictionaryFormatError("file size %d inconsistent with pattern_count %d"
                                        % (len(blob), pc))
        bm = [int(x) for x in np.frombuffer(blob, "<u8", pc, end_table + 4)]
        if any(b2 <= b1 for b1, b2 in zip(bm, bm[1:])):
            raise DictionaryFormatError("canonical bitmaps not strictly ascending")
        return cls(k, table, bm)

    @classmethod
    def load(cls, path) -> "CanonicalDictionary":
        with open(path, "rb") as fh:
            return cls.from_bytes(fh.read())

    def __repr__(self):
        return "CanonicalDictionary(k=%d, patterns=%d)" % (self.k, self.pattern_count)


def _valid_bitmaps(k: int) -> np.ndarray:
    nbits = stored_bits(k)
    out = []
    step = 1 << 22
    for start in range(0, 1 << nbits, step):
        v = np.arange(start, min(start + step, 1 << nbits), dtype=np.uint64)
        ok = np.ones(len(v), dtype=bool)
        for i in range(2, k):
            ok &= ((v >> np.uint64(group_offset(i))) & np.uint64((1 << i) - 1)) != 0
        out.append(v[ok])
    return np.concatenate(out)


_DICT_CACHE: dict = {}


def _build_on_device(k: int) -> CanonicalDictionary:
    """The orbit sweep on the GPU (``wm_dictionary_build``, csrc/wm_dict.cu)."""
    import ctypes
    from . import _native
    table = np.empty(1 << stored_bits(k), dtype=np.uint32)
    reps = np.zeros(1 << 16, dtype=np.uint64)
    count = ctypes.c_uint32()
    _native.check(_native.load().wm_dictionary_build(
        k, table.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
        reps.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(reps), ctypes.byref(count)))
    return CanonicalDictionary(k, table, [int(b) for b in reps[:count.value]])


def build_dictionary(k: int, allow_large: bool = False, device=None) -> CanonicalDictionary:
    """Full pattern dictionary for size ``k`` (reference ``canon.py:315-343``).
    Deterministic; cached per process.  ``device=True`` runs the orbit sweep
    on the GPU (same bytes); ``None`` picks the GPU for k = 8, where the host
    sweep over ~1e8 bitmaps is impractical."""
    if not 3 <= k <= K_MAX_LARGE:
        raise ValueError("dictionary supports 3 <= k <= %d, got k=%d" % (K_MAX_LARGE, k))
    if k > K_MAX_DEFAULT and not allow_large:
        raise ValueError("k=%d needs allow_large=True (2^%d-entry table)" % (k, stored_bits(k)))
    if k in _DICT_CACHE and not device:
        d = _DICT_CACHE[k]
        return CanonicalDictionary(k, d.table.copy(), d.canonical_bitmaps)
    if device is None and k > K_MAX_DEFAULT:
        try:
            import torch
            device = torch.cuda.is_available()
        except ImportError:
            device = False
    if device:
        d = _build_on_device(k)
        _DICT_CACHE.setdefault(k, d)
        return CanonicalDictionary(k, d.table.copy(), d.canonical_bitmaps)
    table = np.full(1 << stored_bits(k), SENTINEL, dtype=np.uint32)
    reps: list = []
    for b in _valid_bitmaps(k).tolist():
        if table[b] != SENTINEL:
            continue
        img, ok = _orbit(b, k)
        table[img[ok]] = len(reps)
        reps.append(b)
    d = CanonicalDictionary(k, table, reps)
    _DICT_CACHE[k] = d
    return CanonicalDictionary(k, table.copy(), reps)
