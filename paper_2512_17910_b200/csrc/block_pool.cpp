// Native block manager: the per-block state of the paged KV pool and its digest index.
//
// Replaces the per-block Python bookkeeping of
//   /root/reference/pkg/src/aloraserve/kv_cache.py:126-326 (BlockPool)
// with the same observable behaviour:
//   lookup   kv_cache.py:154-183  walk the chain from block 0, stop at the first miss, pin hits
//                                 (a pinned free block leaves the free list wherever it sits)
//   allocate kv_cache.py:192-218  pop the least recently released block; an evicted block's digest
//                                 leaves the index only if the index still points at it; atomic
//                                 (nothing is taken when the request cannot be met)
//   publish  kv_cache.py:250-257  full blocks get their digest; the index entry is overwritten
//                                 (last writer wins)
//   release  kv_cache.py:258-270  tail first; a block whose count drops to 0 joins the free list's
//                                 most-recently-released end
//   set_fill kv_cache.py:220-223  fill = clamp(n_tokens - i*B, 0, B) over a request's blocks
// The per-request maps (request id -> owned blocks) stay in Python; every call here is O(blocks
// touched) with no allocation on the lookup path, so one scheduler admission costs one ctypes call.

#include <cstdint>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "../../include/alora_sm100a.h"

namespace {

struct Digest {
  uint64_t lo, hi;
  bool operator==(const Digest& o) const { return lo == o.lo && hi == o.hi; }
};

struct DigestHash {
  size_t operator()(const Digest& d) const { return static_cast<size_t>(d.lo ^ (d.hi * 0x9e3779b97f4a7c15ULL)); }
};

inline Digest load_digest(const uint8_t* p) {
  Digest d;
  std::memcpy(&d.lo, p, 8);
  std::memcpy(&d.hi, p + 8, 8);
  return d;
}

struct Pool {
  int32_t nb, B;
  std::vector<int32_t> ref, fill;
  std::vector<uint8_t> has_hash;
  std::vector<uint8_t> hash;  // [nb][16]
  std::unordered_map<Digest, int32_t, DigestHash> index;
  // free list in release order: head = least recently released (next to evict)
  std::vector<int32_t> prev, next;
  std::vector<uint8_t> in_free;
  int32_t head = -1, tail = -1, n_free = 0;

  Pool(int32_t n, int32_t b)
      : nb(n), B(b), ref(n, 0), fill(n, 0), has_hash(n, 0), hash(static_cast<size_t>(n) * 16, 0), prev(n, -1),
        next(n, -1), in_free(n, 0) {
    index.reserve(static_cast<size_t>(n) * 2);
    for (int32_t i = 0; i < n; ++i) push_back(i);
  }

  void push_back(int32_t b) {
    prev[b] = tail;
    next[b] = -1;
    if (tail >= 0) next[tail] = b; else head = b;
    tail = b;
    in_free[b] = 1;
    ++n_free;
  }

  void unlink(int32_t b) {
    const int32_t p = prev[b], n = next[b];
    if (p >= 0) next[p] = n; else head = n;
    if (n >= 0) prev[n] = p; else tail = p;
    prev[b] = next[b] = -1;
    in_free[b] = 0;
    --n_free;
  }

  bool digest_of(int32_t b, Digest* d) const {
    if (!has_hash[b]) return false;
    *d = load_digest(&hash[static_cast<size_t>(b) * 16]);
    return true;
  }
};

inline Pool* P(void* h) { return static_cast<Pool*>(h); }

}  // namespace

extern "C" {

void* alora_pool_create(int32_t n_blocks, int32_t block_size) {
  if (n_blocks < 1 || block_size < 1) return nullptr;
  try {
    return new Pool(n_blocks, block_size);
  } catch (...) {
    return nullptr;
  }
}

void alora_pool_destroy(void* pool) { delete P(pool); }

int alora_pool_views(void* pool, int32_t** ref, int32_t** fill, uint8_t** has_hash, uint8_t** hash) {
  if (pool == nullptr) return ALORA_EINVAL;
  Pool* p = P(pool);
  if (ref) *ref = p->ref.data();
  if (fill) *fill = p->fill.data();
  if (has_hash) *has_hash = p->has_hash.data();
  if (hash) *hash = p->hash.data();
  return ALORA_OK;
}

int32_t alora_pool_num_free(void* pool) { return pool ? P(pool)->n_free : ALORA_EINVAL; }

int64_t alora_pool_lookup(void* pool, const uint8_t* digests, int64_t n, int32_t* out_ids) {
  if (pool == nullptr || n < 0 || (n > 0 && (digests == nullptr || out_ids == nullptr))) return ALORA_EINVAL;
  Pool* p = P(pool);
  int64_t hits = 0;
  for (; hits < n; ++hits) {
    auto it = p->index.find(load_digest(digests + 16 * hits));
    if (it == p->index.end()) break;
    const int32_t b = it->second;
    if (p->ref[b] == 0) p->unlink(b);
    ++p->ref[b];
    out_ids[hits] = b;
  }
  return hits;
}

int alora_pool_allocate(void* pool, int64_t n, int32_t* out_ids) {
  if (pool == nullptr || n < 0 || (n > 0 && out_ids == nullptr)) return ALORA_EINVAL;
  Pool* p = P(pool);
  if (n > p->n_free) return ALORA_ENOSPC;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t b = p->head;
    if (p->ref[b] != 0) return ALORA_ESTATE;
    p->unlink(b);
    Digest d;
    if (p->digest_of(b, &d)) {
      auto it = p->index.find(d);
      if (it != p->index.end() && it->second == b) p->index.erase(it);
    }
    p->has_hash[b] = 0;
    p->fill[b] = 0;
    p->ref[b] = 1;
    out_ids[i] = b;
  }
  return ALORA_OK;
}

int alora_pool_release(void* pool, const int32_t* ids, int64_t n) {
  if (pool == nullptr || n < 0 || (n > 0 && ids == nullptr)) return ALORA_EINVAL;
  Pool* p = P(pool);
  for (int64_t i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= p->nb) return ALORA_EINVAL;
  for (int64_t i = n - 1; i >= 0; --i) {  // tail first
    const int32_t b = ids[i];
    if (p->ref[b] < 1) return ALORA_ESTATE;
    if (--p->ref[b] == 0) {
      if (p->in_free[b]) return ALORA_ESTATE;
      p->push_back(b);
    }
  }
  return ALORA_OK;
}

int alora_pool_publish(void* pool, const int32_t* ids, const uint8_t* digests, int64_t n) {
  if (pool == nullptr || n < 0 || (n > 0 && (ids == nullptr || digests == nullptr))) return ALORA_EINVAL;
  Pool* p = P(pool);
  for (int64_t i = 0; i < n; ++i) {
    const int32_t b = ids[i];
    if (b < 0 || b >= p->nb) return ALORA_EINVAL;
    if (p->fill[b] != p->B) return ALORA_ESTATE;  // only full blocks carry a digest
    std::memcpy(&p->hash[static_cast<size_t>(b) * 16], digests + 16 * i, 16);
    p->has_hash[b] = 1;
    p->index[load_digest(digests + 16 * i)] = b;
  }
  return ALORA_OK;
}

int alora_pool_set_fill(void* pool, const int32_t* ids, int64_t n, int64_t first, int64_t n_tokens) {
  if (pool == nullptr || n < 0 || first < 0 || (n > 0 && ids == nullptr)) return ALORA_EINVAL;
  Pool* p = P(pool);
  for (int64_t j = 0; j < n; ++j) {  // ids[j] holds positions [(first+j)*B, (first+j+1)*B)
    const int32_t b = ids[j];
    if (b < 0 || b >= p->nb) return ALORA_EINVAL;
    int64_t f = n_tokens - (first + j) * p->B;
    p->fill[b] = static_cast<int32_t>(f < 0 ? 0 : (f > p->B ? p->B : f));
  }
  return ALORA_OK;
}

int64_t alora_pool_free_list(void* pool, int32_t* out, int64_t cap) {
  if (pool == nullptr || (cap > 0 && out == nullptr)) return ALORA_EINVAL;
  Pool* p = P(pool);
  int64_t k = 0;
  for (int32_t b = p->head; b >= 0 && k < cap; b = p->next[b]) out[k++] = b;
  return k;
}

int32_t alora_pool_index_get(void* pool, const uint8_t* digest) {
  if (pool == nullptr || digest == nullptr) return ALORA_EINVAL;
  auto it = P(pool)->index.find(load_digest(digest));
  return it == P(pool)->index.end() ? -1 : it->second;
}

int64_t alora_pool_index_dump(void* pool, uint8_t* digests, int32_t* ids, int64_t cap) {
  if (pool == nullptr) return ALORA_EINVAL;
  Pool* p = P(pool);
  if (cap <= 0) return static_cast<int64_t>(p->index.size());
  int64_t k = 0;
  for (const auto& kv : p->index) {
    if (k >= cap) break;
    std::memcpy(digests + 16 * k, &kv.first.lo, 8);
    std::memcpy(digests + 16 * k + 8, &kv.first.hi, 8);
    ids[k++] = kv.second;
  }
  return k;
}

}  // extern "C"
