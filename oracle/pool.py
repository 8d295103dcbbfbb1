"""Oracle: KV page allocator and page migration semantics — TEST INFRASTRUCTURE ONLY.

  PAPER.md:281  "the Coordinator consults the scheduler to extract sequence
                metadata (e.g., token count, KV cache location and size),
                allocates memory on the target instance, and transfers the KV cache"
  PAPER.md:428  "KV caches are transferred directly into idle slots on the target
                instance, and migration is skipped if no idle cache is available."

Readings: Z26 whole pages ceil(L/16) are copied; Z27 destination
pages are the lowest free page indices, all-or-nothing; Z28 no idle cache ->
NO_PAGES with the pool unchanged; double free is an error.
"""
from __future__ import annotations

import numpy as np


class NoPages(Exception):
    pass


class InvalidFree(Exception):
    pass


class PagePool:
    """Deterministic lowest-free-first allocator over pages 0..num_pages-1."""

    def __init__(self, num_pages: int):
        if num_pages < 0:
            raise ValueError("num_pages must be >= 0")
        self.num_pages = int(num_pages)
        self.free = [True] * self.num_pages

    def num_free(self) -> int:
        return sum(self.free)

    def alloc(self, n: int):
        """The n lowest free page ids in ascending order, or NoPages (pool unchanged)."""
        if n < 0:
            raise ValueError("n must be >= 0")
        out = []
        for p in range(self.num_pages):
            if len(out) == n:
                break
            if self.free[p]:
                out.append(p)
        if len(out) < n:
            raise NoPages(f"need {n}, have {len(out)}")
        for p in out:
            self.free[p] = False
        return out

    def release(self, pages):
        """Free pages; freeing a page that is not allocated (or twice) is an error
        and leaves the pool unchanged."""
        pages = [int(p) for p in pages]
        seen = set()
        for p in pages:
            if p < 0 or p >= self.num_pages or self.free[p] or p in seen:
                raise InvalidFree(f"page {p}")
            seen.add(p)
        for p in pages:
            self.free[p] = True


def migrate(src_k, src_v, src_pages, dst_k, dst_v, dst_pool: PagePool):
    """One request's pages src -> dst (numpy pools [layers?, num_pages, ...]).

    Allocates len(src_pages) destination pages from dst_pool (Z27), then copies
    whole pages (Z26).  Returns the destination page list.  On NoPages nothing
    is copied and the pool is unchanged (Z28)."""
    dst_pages = dst_pool.alloc(len(src_pages))
    sp = np.asarray(src_pages, dtype=np.int64)
    dp = np.asarray(dst_pages, dtype=np.int64)
    dst_k[..., dp, :, :, :] = src_k[..., sp, :, :, :]
    dst_v[..., dp, :, :, :] = src_v[..., sp, :, :, :]
    return dst_pages
