"""ORACLE -- CPU restatement of the device KV pool.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may import this module, and only as the checker or the
CPU baseline -- never as the product path.

What it restates.  The reference (pkg/src/dropsim/memory.py) is
token-granular and position-free: its KVAllocator counts tokens against
`kvcache_virtual_extent`, `drop_layers` grows the extent by whole layer
blocks (memory.py:147-172) and `restore_layers` reserves bytes before the
extent shrinks (memory.py:175-197, 116-124).  The device adds pages and
block tables underneath (csrc/kb_pool.cu); this module restates that device
layer with the same deterministic rules, so block tables, owners and moved
bytes can be compared bit for bit:
  * page space: [head pages | slab of layer 0 | ... | slab of layer L-1];
    a held layer's slab pages are reserved (they hold its weights);
  * drop(lo, hi): the slab pages of layers [lo, hi) become free KV pages;
  * grow: the K lowest free page ids, assigned in request order, then layer
    order, then page order;
  * release: every page of (slot, layer in [lo, hi)) goes back to the pool;
  * restore(lo, hi): refused unless every live page fits outside the slabs
    of [lo, hi); otherwise their live pages move, in ascending order, to the
    lowest free pages outside the range (compaction) and the range is
    reserved again for the parameter pull.
Page contents are optional numpy byte arrays (small configs only) so copies
and appends can be checked byte for byte.

Parity pinning: the token-level counters this layer sits under are pinned
against the reference's own outputs (tests/golden/memory_ops.json, produced
by tests/golden/make_golden.py from pkg/src/dropsim); page ids and page
bytes have no reference counterpart (page/block-table layout
is unpinned at the reference level) and are pinned by the rules above, which
tests/test_oracle.py checks against brute-force invariants.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

RESERVED = -2  # owner id of a page that holds live weights


@dataclass
class OraclePool:
    num_layers: int
    slab_bytes: int
    page_bytes: int
    head_pages: int            # slack + residual pages mapped at creation
    max_slots: int
    max_pages_per_seq: int
    track_bytes: bool = False
    live: np.ndarray = field(init=False)
    reserved: np.ndarray = field(init=False)
    owner: dict = field(init=False)
    bt: dict = field(init=False)       # (slot, layer) -> list of page ids
    data: Optional[np.ndarray] = field(init=False, default=None)

    def __post_init__(self):
        assert self.slab_bytes % self.page_bytes == 0
        self.slab_pages = self.slab_bytes // self.page_bytes
        self.max_pages = self.head_pages + self.num_layers * self.slab_pages
        self.live = np.zeros(self.max_pages, dtype=bool)
        self.reserved = np.zeros(self.max_pages, dtype=bool)
        self.reserved[self.head_pages:] = True
        self.owner = {}
        self.bt = {}
        if self.track_bytes:
            self.data = np.zeros((self.max_pages, self.page_bytes), dtype=np.uint8)

    def slab_range(self, lo: int, hi: int) -> tuple[int, int]:
        return self.head_pages + lo * self.slab_pages, self.head_pages + hi * self.slab_pages

    # cell id exactly as the device encodes owner[] (csrc/kb_pool.cu grow_kernel)
    def cell(self, slot: int, layer: int, idx: int) -> int:
        return (slot * self.num_layers + layer) * self.max_pages_per_seq + idx

    def npages(self, slot: int, layer: int) -> int:
        return len(self.bt.get((slot, layer), ()))

    @property
    def live_pages(self) -> int:
        return int(self.live.sum())

    @property
    def usable_pages(self) -> int:
        return int((~self.reserved).sum())

    def free_pages(self) -> np.ndarray:
        return np.flatnonzero(~(self.live | self.reserved))

    def grow(self, reqs) -> bool:
        need = sum((hi - lo) * add for _, lo, hi, add in reqs)
        free = self.free_pages()
        if need > len(free):
            return False
        k = 0
        for slot, lo, hi, add in reqs:
            for layer in range(lo, hi):
                row = self.bt.setdefault((slot, layer), [])
                for _ in range(add):
                    page = int(free[k])
                    k += 1
                    self.owner[page] = self.cell(slot, layer, len(row))
                    row.append(page)
                    self.live[page] = True
        return True

    def release(self, slots, lo: int, hi: int) -> None:
        for slot in slots:
            for layer in range(lo, hi):
                for page in self.bt.pop((slot, layer), []):
                    self.live[page] = False
                    self.owner.pop(page, None)

    def drop(self, lo: int, hi: int) -> None:
        a, b = self.slab_range(lo, hi)
        assert self.reserved[a:b].all()
        self.reserved[a:b] = False

    def restore(self, lo: int, hi: int) -> int:
        """Vacate the slabs of [lo, hi); returns pages moved, or -1 if refused."""
        a, b = self.slab_range(lo, hi)
        assert not self.reserved[a:b].any()
        if self.live_pages > self.usable_pages - (b - a):
            return -1
        src = np.flatnonzero(self.live[a:b]) + a
        free = self.free_pages()
        dst = free[(free < a) | (free >= b)][:len(src)]
        assert len(dst) == len(src)
        for s, d in zip(src.tolist(), dst.tolist()):
            cell = self.owner.pop(s)
            slot_layer, idx = divmod(cell, self.max_pages_per_seq)
            slot, layer = divmod(slot_layer, self.num_layers)
            self.bt[(slot, layer)][idx] = d
            self.owner[d] = cell
            self.live[s] = False
            self.live[d] = True
            if self.data is not None:
                self.data[d] = self.data[s]
        self.reserved[a:b] = True
        return len(src)

    def owner_array(self) -> np.ndarray:
        """owner[] as the device stores it: cell, -2 reserved, -1 free."""
        out = np.full(self.max_pages, -1, dtype=np.int32)
        out[self.reserved] = RESERVED
        for pg, cell in self.owner.items():
            out[pg] = cell
        return out

    def bitmap(self) -> np.ndarray:
        return self.live | self.reserved


def copy_pages(dst: OraclePool, src: OraclePool, moves) -> int:
    """Byte copy of the flattened page ranges (csrc/kb_copy.cu copy_pages_kernel).
    Returns bytes moved."""
    moved = 0
    for s_slot, d_slot, lo, hi, npages, flo, fhi in moves:
        for flat in range(flo, fhi):
            layer = lo + flat // npages
            idx = flat % npages
            sp = src.bt[(s_slot, layer)][idx]
            dp = dst.bt[(d_slot, layer)][idx]
            dst.data[dp] = src.data[sp]
            moved += src.page_bytes
    return moved


def bf16_bits_to_f16_bits(x: np.ndarray) -> np.ndarray:
    """bf16 bit patterns -> fp16 bit patterns, round-to-nearest-even (what
    __floats2half2_rn does in csrc/kb_append.cu); out-of-range values
    saturate to inf / flush like the device (which also flags them)."""
    f = (np.asarray(x, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)
    with np.errstate(over="ignore", under="ignore"):
        return f.astype(np.float16).view(np.uint16)


def v_range_flags(v_bits: np.ndarray) -> int:
    """KB_KV_V_OVERFLOW (1) / KB_KV_V_UNDERFLOW (2) for bf16 V bit patterns
    [..., head_dim] (csrc/kb_append.cu): any |v| >= 2^16 (inf / NaN
    included), or a row (one token, one kv head) whose largest magnitude is
    nonzero and below 2^-14."""
    m = np.asarray(v_bits, dtype=np.uint16).astype(np.uint32) & 0x7FFF
    flags = 0
    if (m >= 0x4780).any():
        flags |= 1
    rmax = m.max(axis=-1)
    if ((rmax > 0) & (rmax < 0x3880)).any():
        flags |= 2
    return flags


_PHI = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _fmix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def hash_bytes(buf) -> int:
    """Position-sensitive 64-bit content hash of one segment
    (csrc/kb_hash.cu kb_hash_segments): fmix(S ^ nbytes) with
    S = sum_j fmix(w_j ^ j * phi) mod 2^64 over little-endian uint64 words."""
    a = np.frombuffer(bytes(buf) if not isinstance(buf, np.ndarray) else buf.tobytes(),
                      dtype="<u8")
    with np.errstate(over="ignore"):
        idx = np.arange(a.size, dtype=np.uint64) * _PHI
        s = np.sum(_fmix64(a ^ idx), dtype=np.uint64)
    h = _fmix64(np.array([s ^ np.uint64(a.size * 8)], dtype=np.uint64))[0]
    return int(h.astype(np.int64))  # as the device's int64 view


def kv_append(pool: OraclePool, layer: int, k: np.ndarray, v: np.ndarray, slots, pos,
              n_kv_heads: int, block_tokens: int, head_dim: int = 128) -> None:
    """Scatter K/V rows into pages laid out [K|V][kv_head][token][head_dim]
    (csrc/kb_append.cu): K stored as given (bf16), V converted to fp16.
    k, v: uint16 bf16 bit patterns [ntok, n_kv_heads, head_dim]."""
    row_bytes = head_dim * 2
    half = pool.page_bytes // 2
    for t in range(k.shape[0]):
        page = pool.bt[(int(slots[t]), layer)][int(pos[t]) // block_tokens]
        r = int(pos[t]) % block_tokens
        buf = pool.data[page]
        for h in range(n_kv_heads):
            off = (h * block_tokens + r) * row_bytes
            buf[off:off + row_bytes] = k[t, h].view(np.uint8)
            buf[half + off:half + off + row_bytes] = bf16_bits_to_f16_bits(v[t, h]).view(np.uint8)


def gather_kv(pool: OraclePool, slot: int, layer: int, ctx: int, n_kv_heads: int,
              block_tokens: int, head_dim: int = 128):
    """K (bf16 bits), V (fp16 bits) of the first ctx tokens as uint16 arrays
    [ctx, n_kv_heads, head_dim]."""
    half = pool.page_bytes // 2
    k = np.zeros((ctx, n_kv_heads, head_dim), dtype=np.uint16)
    v = np.zeros_like(k)
    row = pool.bt[(slot, layer)]
    for t in range(ctx):
        page = pool.data[row[t // block_tokens]]
        r = t % block_tokens
        for h in range(n_kv_heads):
            off = (h * block_tokens + r) * head_dim * 2
            k[t, h] = page[off:off + head_dim * 2].view(np.uint16)
            v[t, h] = page[half + off:half + off + head_dim * 2].view(np.uint16)
    return k, v
