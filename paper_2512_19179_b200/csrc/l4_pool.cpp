// Host-side KV page pool: deterministic lowest-free-first allocator (Z27).
//
// P:428 "KV caches are transferred directly into idle slots on the target
// instance, and migration is skipped if no idle cache is available."  The pool
// is the bookkeeping of those idle slots: a bitset of free pages scanned from
// the lowest word, all-or-nothing allocation (NO_PAGES leaves it unchanged,
// Z28) and checked frees (double free -> INVALID_ARG, nothing changed).
#include <algorithm>
#include <cstring>
#include <new>
#include <vector>

#include "l4_internal.h"

struct l4_page_pool {
  int64_t num_pages = 0;
  int64_t num_free = 0;
  std::vector<uint64_t> free_bits;  // bit set = page free
};

extern "C" l4_status l4_pool_create(int64_t num_pages, l4_page_pool** out) {
  L4_CHECK_ARG(out != nullptr, "l4_pool_create: out is NULL");
  L4_CHECK_ARG(num_pages >= 0 && num_pages <= (int64_t)INT32_MAX, "l4_pool_create: num_pages out of range");
  l4_page_pool* p = new (std::nothrow) l4_page_pool();
  if (!p) return l4::fail(L4_ERR_INVALID_ARG, "l4_pool_create: out of host memory");
  p->num_pages = num_pages;
  p->num_free = num_pages;
  p->free_bits.assign((size_t)((num_pages + 63) / 64), ~0ull);
  if (num_pages % 64) p->free_bits.back() = (1ull << (num_pages % 64)) - 1;
  *out = p;
  return L4_OK;
}

extern "C" l4_status l4_pool_alloc(l4_page_pool* pool, int64_t n, int32_t* pages_out) {
  L4_CHECK_ARG(pool != nullptr, "l4_pool_alloc: pool is NULL");
  L4_CHECK_ARG(n >= 0, "l4_pool_alloc: n < 0");
  L4_CHECK_ARG(n == 0 || pages_out != nullptr, "l4_pool_alloc: pages_out is NULL");
  if (n > pool->num_free) {
    l4::set_error("l4_pool_alloc: need %lld pages, %lld free", (long long)n, (long long)pool->num_free);
    return L4_ERR_NO_PAGES;
  }
  int64_t got = 0;
  for (size_t w = 0; w < pool->free_bits.size() && got < n; ++w) {
    uint64_t bits = pool->free_bits[w];
    while (bits && got < n) {
      int b = __builtin_ctzll(bits);
      bits &= bits - 1;
      pages_out[got++] = (int32_t)(w * 64 + b);
    }
  }
  for (int64_t i = 0; i < n; ++i) {
    int64_t p = pages_out[i];
    pool->free_bits[p >> 6] &= ~(1ull << (p & 63));
  }
  pool->num_free -= n;
  return L4_OK;
}

extern "C" l4_status l4_pool_free(l4_page_pool* pool, const int32_t* pages, int64_t n) {
  L4_CHECK_ARG(pool != nullptr, "l4_pool_free: pool is NULL");
  L4_CHECK_ARG(n >= 0, "l4_pool_free: n < 0");
  L4_CHECK_ARG(n == 0 || pages != nullptr, "l4_pool_free: pages is NULL");
  std::vector<int32_t> sorted(pages, pages + n);
  std::sort(sorted.begin(), sorted.end());
  for (int64_t i = 0; i < n; ++i) {
    int64_t p = sorted[i];
    if (p < 0 || p >= pool->num_pages) {
      l4::set_error("l4_pool_free: page %lld out of range", (long long)p);
      return L4_ERR_INVALID_ARG;
    }
    if (i > 0 && sorted[i - 1] == p) {
      l4::set_error("l4_pool_free: page %lld repeated", (long long)p);
      return L4_ERR_INVALID_ARG;
    }
    if (pool->free_bits[p >> 6] & (1ull << (p & 63))) {
      l4::set_error("l4_pool_free: page %lld is not allocated", (long long)p);
      return L4_ERR_INVALID_ARG;
    }
  }
  for (int64_t i = 0; i < n; ++i) {
    int64_t p = sorted[i];
    pool->free_bits[p >> 6] |= (1ull << (p & 63));
  }
  pool->num_free += n;
  return L4_OK;
}

extern "C" int64_t l4_pool_num_free(const l4_page_pool* pool) { return pool ? pool->num_free : -1; }

extern "C" void l4_pool_destroy(l4_page_pool* pool) { delete pool; }
