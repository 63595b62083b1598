// Native admission: the continuous-batching scheduler and the per-request block tables of the engine.
//
// Replaces, with the same observable behaviour (hits, spans, stamps, traces, pool digests):
//   /root/reference/pkg/src/aloraserve/scheduler.py:139-158   thread-safe intake, ticket order
//   scheduler.py:160-212   schedule_step: decodes first (one token each while budget and batch slots
//                          last; a decode that cannot get its next block fails the request), then prefills
//                          strictly FCFS (running, then waiting), chunk = min(remaining, budget), a deferred
//                          head blocks everyone behind it
//   scheduler.py:215-235   one prefix lookup per request at its first scheduling, hit tokens count as
//                          processed; _ensure_blocks allocates the blocks a span needs (atomic, LRU)
//   scheduler.py:247-265   on_span_done: processed / computed / generated, PREFILLING -> DECODING when the
//                          prompt completes, FINISHED at max_new_tokens
//   kv_cache.py:154-183, 192-218, 220-223, 234-271  lookup walk, allocate, set_fill, commit_and_free / release
//                          (the per-block state is the native block manager of block_pool.cpp)
// One engine step is one call: the step's lookup chains are hashed in one batch (alora_hash_requests, shared
// base prefixes hashed once), the spans and each span's block table come back in flat arrays, and the step's
// completions are applied in one call. The Python Engine keeps the Request objects for the clock stamps and
// metrics (engine.py / metrics.py) and mirrors the counters this core returns.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/alora_sm100a.h"

namespace {

enum State : int32_t { kQueued = 0, kPrefilling = 1, kDecoding = 2, kFinished = 3 };
enum Mode : int32_t { kBase = 0, kStandard = 1, kActivated = 2 };

struct Req {
  std::vector<int64_t> tok;  // prompt, then generated tokens (placeholders until set_token)
  int64_t prompt_len = 0;
  int32_t max_new = 0;
  int64_t processed = 0, computed = 0, hit = 0;
  int32_t n_gen = 0;
  int32_t state = kQueued;
  int32_t mode = kBase;
  int64_t inv_start = -1;
  std::string key;
  bool cache_checked = false, failed = false, alive = true, retired = false;
  std::vector<int32_t> blocks;
  int32_t n_reused = 0;
  int64_t filled = 0;
  std::vector<uint8_t> chain;  // admission lookup digests (limit blocks), reused by the commit
};

struct Core {
  void* pool;
  int32_t B, budget, max_batch, hash_threads;
  bool chunked, prefix_caching;
  std::vector<Req> reqs;
  std::mutex intake_mu;
  std::vector<std::vector<int64_t>> spare_tok;  // token buffers of retired requests (<= 256), reused by submit
  std::vector<int32_t> intake;  // handles in submit (ticket) order
  std::deque<int32_t> waiting;
  std::vector<int32_t> prefilling, decoding;
  std::vector<int32_t> scratch;
  // blocks [0, base_blocks) of an n_blocks sequence carry the base key "" (compute_block_keys, kv_cache.py:72-96)
  int64_t base_blocks(const Req& r, int64_t n_blocks) const {
    if (r.mode == kBase) return n_blocks;
    if (r.mode == kStandard) return 0;
    return std::min<int64_t>(n_blocks, r.inv_start / B);
  }
};

inline Core* C(void* h) { return static_cast<Core*>(h); }

bool ensure_blocks(Core& c, Req& r, int64_t n_tokens) {
  const int64_t need = (n_tokens + c.B - 1) / c.B - static_cast<int64_t>(r.blocks.size());
  if (need <= 0) return true;
  c.scratch.resize(static_cast<size_t>(need));
  const int rc = alora_pool_allocate(c.pool, need, c.scratch.data());
  if (rc != ALORA_OK) return false;  // ALORA_ENOSPC: nothing was taken
  r.blocks.insert(r.blocks.end(), c.scratch.begin(), c.scratch.end());
  return true;
}

void remove_from(std::vector<int32_t>& v, int32_t h) {
  auto it = std::find(v.begin(), v.end(), h);
  if (it != v.end()) v.erase(it);
}

// the lookup chains of every request this step may admit, hashed in one batch (scheduler._prehash)
void prehash(Core& c, int64_t n_max) {
  std::vector<int32_t> todo;
  for (int32_t h : c.waiting) {
    if (static_cast<int64_t>(todo.size()) >= n_max) break;
    Req& r = c.reqs[h];
    if (!r.cache_checked && r.chain.empty()) todo.push_back(h);
  }
  if (todo.empty()) return;
  std::vector<const int64_t*> toks;
  std::vector<int64_t> nb, nbase;
  std::vector<const char*> keys;
  std::vector<int32_t> klen;
  int64_t total = 0;
  for (int32_t h : todo) {
    Req& r = c.reqs[h];
    const int64_t limit = std::max<int64_t>(0, (r.prompt_len - 1) / c.B);
    toks.push_back(r.tok.data());
    nb.push_back(limit);
    nbase.push_back(c.base_blocks(r, (r.prompt_len + c.B - 1) / c.B));
    keys.push_back(r.key.c_str());
    klen.push_back(static_cast<int32_t>(r.key.size()));
    total += limit;
  }
  std::vector<uint8_t> out(static_cast<size_t>(std::max<int64_t>(1, total)) * 16);
  if (alora_hash_requests(static_cast<int32_t>(todo.size()), toks.data(), nb.data(), nbase.data(), keys.data(),
                          klen.data(), c.B, out.data(), c.hash_threads) != ALORA_OK)
    return;  // the per-request path below hashes (and reports) on its own
  int64_t off = 0;
  for (size_t i = 0; i < todo.size(); ++i) {
    Req& r = c.reqs[todo[i]];
    r.chain.assign(out.begin() + off * 16, out.begin() + (off + nb[i]) * 16);
    off += nb[i];
  }
}

int cache_lookup(Core& c, Req& r) {
  if (c.prefix_caching) {
    const int64_t limit = std::max<int64_t>(0, (r.prompt_len - 1) / c.B);
    if (static_cast<int64_t>(r.chain.size()) != limit * 16) {
      const int64_t* tp = r.tok.data();
      const char* kp = r.key.c_str();
      const int32_t kl = static_cast<int32_t>(r.key.size());
      const int64_t nbase = c.base_blocks(r, (r.prompt_len + c.B - 1) / c.B);
      r.chain.assign(static_cast<size_t>(std::max<int64_t>(1, limit)) * 16, 0);
      const int rc = alora_hash_requests(1, &tp, &limit, &nbase, &kp, &kl, c.B, r.chain.data(), 1);
      if (rc != ALORA_OK) return rc;
      r.chain.resize(static_cast<size_t>(limit) * 16);
    }
    r.blocks.resize(static_cast<size_t>(limit));
    const int64_t n = limit ? alora_pool_lookup(c.pool, r.chain.data(), limit, r.blocks.data()) : 0;
    if (n < 0) return static_cast<int>(n);
    r.blocks.resize(static_cast<size_t>(n));
    r.hit = n * c.B;
  } else {
    r.blocks.clear();
    r.hit = 0;
  }
  r.n_reused = static_cast<int32_t>(r.blocks.size());
  r.filled = r.hit;  // cached blocks are full: fill bookkeeping starts after them
  r.processed = r.hit;
  r.cache_checked = true;
  return ALORA_OK;
}

int set_fill(Core& c, Req& r) {
  const int64_t first = r.processed >= r.filled ? r.filled / c.B : 0;
  if (first < static_cast<int64_t>(r.blocks.size())) {
    const int rc = alora_pool_set_fill(c.pool, r.blocks.data() + first,
                                       static_cast<int64_t>(r.blocks.size()) - first, first, r.processed);
    if (rc != ALORA_OK) return rc;
  }
  r.filled = r.processed;
  return ALORA_OK;
}

// commit_and_free (kv_cache.py:234-261): publish every full block of the processed tokens, release tail first
int commit(Core& c, Req& r) {
  const int64_t n = r.processed;
  if (static_cast<int64_t>(r.blocks.size()) != (n + c.B - 1) / c.B) return ALORA_ESTATE;
  const int64_t n_full = n / c.B;
  if (n_full > 0) {
    std::vector<uint8_t> dg(static_cast<size_t>(n_full) * 16);
    const int64_t head = std::min<int64_t>(static_cast<int64_t>(r.chain.size()) / 16, n_full);
    // the admission chain covers the unchanged prompt prefix with the same keys (blocks below inv_start / B
    // carry "" whatever the sequence length)
    std::memcpy(dg.data(), r.chain.data(), static_cast<size_t>(head) * 16);
    if (head < n_full) {
      const int64_t nb = n_full - head;
      std::vector<uint32_t> t32(static_cast<size_t>(nb * c.B));
      for (int64_t i = 0; i < nb * c.B; ++i) {
        const int64_t v = r.tok[static_cast<size_t>(head * c.B + i)];
        if (v < 0 || v > 0xffffffffLL) return ALORA_EINVAL;
        t32[static_cast<size_t>(i)] = static_cast<uint32_t>(v);
      }
      const int64_t nbase = c.base_blocks(r, (n + c.B - 1) / c.B);
      std::string blob;
      std::vector<int64_t> off(static_cast<size_t>(nb) + 1, 0);
      for (int64_t i = 0; i < nb; ++i) {
        const bool base = head + i < nbase;
        if (!base) blob += r.key;
        off[static_cast<size_t>(i) + 1] = static_cast<int64_t>(blob.size());
      }
      if (blob.empty()) blob.push_back('\0');
      const int rc = alora_hash_chain(head > 0 ? dg.data() + (head - 1) * 16 : nullptr, t32.data(), nb, c.B,
                                      blob.data(), off.data(), dg.data() + head * 16);
      if (rc != ALORA_OK) return rc;
    }
    const int rc = alora_pool_publish(c.pool, r.blocks.data(), dg.data(), n_full);
    if (rc != ALORA_OK) return rc;
  }
  const int rc = alora_pool_release(c.pool, r.blocks.data(), static_cast<int64_t>(r.blocks.size()));
  r.blocks.clear();
  return rc;
}

}  // namespace

extern "C" {

void* alora_sched_create(void* pool, int32_t block_size, int32_t token_budget, int32_t max_batch, int32_t chunked,
                         int32_t prefix_caching, int32_t hash_threads) {
  if (!pool || block_size < 1 || token_budget < 1 || max_batch < 1) return nullptr;
  Core* c = new (std::nothrow) Core();
  if (!c) return nullptr;
  c->pool = pool;
  c->B = block_size;
  c->budget = token_budget;
  c->max_batch = max_batch;
  c->chunked = chunked != 0;
  c->prefix_caching = prefix_caching != 0;
  c->hash_threads = std::max(1, hash_threads);
  return c;
}

void alora_sched_destroy(void* s) { delete C(s); }

int32_t alora_sched_submit(void* s, const int64_t* prompt, int64_t n, int32_t max_new, int32_t mode, const char* key,
                           int32_t key_len, int64_t inv_start) {
  if (!s || !prompt || n < 1 || max_new < 1 || mode < kBase || mode > kActivated || key_len < 0) return ALORA_EINVAL;
  if (mode == kActivated && (inv_start < 0 || inv_start > n)) return ALORA_EINVAL;
  Core& c = *C(s);
  Req r;
  {  // a retired request's token buffer when one is parked (no fresh pages on the submit path)
    std::lock_guard<std::mutex> l(c.intake_mu);
    if (!c.spare_tok.empty()) {
      r.tok = std::move(c.spare_tok.back());
      c.spare_tok.pop_back();
    }
  }
  r.tok.reserve(static_cast<size_t>(n + max_new));  // one allocation for the prompt and every generated token
  r.tok.assign(prompt, prompt + n);
  r.prompt_len = n;
  r.max_new = max_new;
  r.mode = mode;
  r.inv_start = inv_start;
  if (mode != kBase && key_len > 0) r.key.assign(key, key + key_len);
  std::lock_guard<std::mutex> l(c.intake_mu);  // intake is thread-safe; the step loop is single-threaded
  c.reqs.push_back(std::move(r));
  const int32_t h = static_cast<int32_t>(c.reqs.size()) - 1;
  c.intake.push_back(h);
  return h;
}

int32_t alora_sched_has_work(void* s) {
  if (!s) return ALORA_EINVAL;
  Core& c = *C(s);
  std::lock_guard<std::mutex> l(c.intake_mu);
  return (!c.intake.empty() || !c.waiting.empty() || !c.prefilling.empty() || !c.decoding.empty()) ? 1 : 0;
}

int alora_sched_step(void* s, int32_t* spans, int32_t span_cap, int32_t* failed, int32_t failed_cap,
                     int32_t* looked, int32_t looked_cap, int32_t* counts, int32_t* blocks, int64_t block_cap,
                     int64_t* block_off) {
  if (!s || !spans || !failed || !looked || !counts || !blocks || !block_off || span_cap < 1) return ALORA_EINVAL;
  Core& c = *C(s);
  {
    std::lock_guard<std::mutex> l(c.intake_mu);
    for (int32_t h : c.intake) c.waiting.push_back(h);
    c.intake.clear();
  }
  int64_t budget = c.budget;
  int32_t n_spans = 0, n_failed = 0, n_looked = 0;
  int64_t used = 0;
  auto emit = [&](int32_t h, int64_t a, int64_t b, int32_t kind) {
    if (n_spans >= span_cap) return false;
    spans[4 * n_spans] = h;
    spans[4 * n_spans + 1] = static_cast<int32_t>(a);
    spans[4 * n_spans + 2] = static_cast<int32_t>(b);
    spans[4 * n_spans + 3] = kind;
    ++n_spans;
    used += b - a;
    return true;
  };
  // decodes first, one token each (scheduler.py:174-184)
  const std::vector<int32_t> dec = c.decoding;
  for (int32_t h : dec) {
    if (budget == 0 || n_spans >= c.max_batch) break;
    Req& r = c.reqs[h];
    if (!ensure_blocks(c, r, r.processed + 1)) {
      r.failed = true;
      r.state = kFinished;
      remove_from(c.decoding, h);
      remove_from(c.prefilling, h);
      if (n_failed < failed_cap) failed[n_failed++] = h;
      continue;
    }
    if (!emit(h, r.processed, r.processed + 1, 1)) return ALORA_EINVAL;
    budget -= 1;
  }
  if (c.prefix_caching) prehash(c, c.max_batch - n_spans);
  // prefills strictly FCFS: running prefills, then the waiting queue (scheduler.py:186-210)
  std::vector<int32_t> order(c.prefilling.begin(), c.prefilling.end());
  order.insert(order.end(), c.waiting.begin(), c.waiting.end());
  for (int32_t h : order) {
    if ((budget == 0 && c.chunked) || n_spans >= c.max_batch) break;
    Req& r = c.reqs[h];
    if (!r.cache_checked) {
      const int rc = cache_lookup(c, r);
      if (rc != ALORA_OK) return rc;
      if (n_looked < looked_cap) looked[n_looked++] = h;
    }
    const int64_t remaining = r.prompt_len - r.processed;
    if (remaining <= 0) return ALORA_ESTATE;
    const int64_t chunk = c.chunked ? std::min(remaining, budget) : remaining;
    if (chunk == 0 || !ensure_blocks(c, r, r.processed + chunk)) break;
    int32_t kind = 0;
    if (r.state == kQueued) {
      kind |= 256;  // first scheduled work: the prefill_start stamp
      r.state = kPrefilling;
      auto it = std::find(c.waiting.begin(), c.waiting.end(), h);
      if (it != c.waiting.end()) c.waiting.erase(it);
      c.prefilling.push_back(h);
    }
    if (!emit(h, r.processed, r.processed + chunk, kind)) return ALORA_EINVAL;
    budget = std::max<int64_t>(0, budget - chunk);
    if (!c.chunked) break;
  }
  // each span's block table (the request's owned ids in position order)
  int64_t off = 0;
  for (int32_t i = 0; i < n_spans; ++i) {
    const Req& r = c.reqs[spans[4 * i]];
    block_off[i] = off;
    if (off + static_cast<int64_t>(r.blocks.size()) > block_cap) return ALORA_EINVAL;
    std::memcpy(blocks + off, r.blocks.data(), r.blocks.size() * sizeof(int32_t));
    off += static_cast<int64_t>(r.blocks.size());
  }
  block_off[n_spans] = off;
  counts[0] = n_spans;
  counts[1] = n_failed;
  counts[2] = n_looked;
  counts[3] = static_cast<int32_t>(used);
  return ALORA_OK;
}

int alora_sched_step_done(void* s, int32_t n, const int32_t* handles, const int32_t* starts, const int32_t* ends,
                          const int64_t* emitted, const uint8_t* has_emitted, uint8_t* flags_out) {
  if (!s || n < 0 || (n > 0 && (!handles || !starts || !ends || !emitted || !has_emitted || !flags_out)))
    return ALORA_EINVAL;
  Core& c = *C(s);
  for (int32_t i = 0; i < n; ++i) {
    Req& r = c.reqs[handles[i]];
    if (starts[i] != r.processed || ends[i] < starts[i]) return ALORA_ESTATE;
    r.processed = ends[i];
    r.computed += ends[i] - starts[i];
    uint8_t f = 0;
    if (has_emitted[i]) {
      r.tok.push_back(emitted[i]);
      ++r.n_gen;
    }
    if (r.state == kPrefilling && r.processed == r.prompt_len) {
      r.state = kDecoding;
      remove_from(c.prefilling, handles[i]);
      c.decoding.push_back(handles[i]);
      f |= 1;
    }
    if (r.n_gen >= r.max_new) {
      r.state = kFinished;
      remove_from(c.decoding, handles[i]);
      f |= 2;
    }
    const int rc = set_fill(c, r);
    if (rc != ALORA_OK) return rc;
    flags_out[i] = f;
  }
  return ALORA_OK;
}

int alora_sched_set_token(void* s, int32_t h, int64_t gen_index, int64_t token) {
  if (!s || h < 0 || h >= static_cast<int32_t>(C(s)->reqs.size())) return ALORA_EINVAL;
  Req& r = C(s)->reqs[h];
  if (gen_index < 0 || gen_index >= r.n_gen) return ALORA_EINVAL;
  r.tok[static_cast<size_t>(r.prompt_len + gen_index)] = token;
  return ALORA_OK;
}

int alora_sched_retire(void* s, int32_t h) {
  if (!s || h < 0 || h >= static_cast<int32_t>(C(s)->reqs.size())) return ALORA_EINVAL;
  Core& c = *C(s);
  Req& r = c.reqs[h];
  if (r.retired) return ALORA_ESTATE;
  r.retired = true;
  int rc = ALORA_OK;
  if (r.failed) {
    rc = alora_pool_release(c.pool, r.blocks.data(), static_cast<int64_t>(r.blocks.size()));
    r.blocks.clear();
  } else {
    rc = commit(c, r);
  }
  r.chain.clear();
  r.chain.shrink_to_fit();
  {  // the Python Request keeps the tokens; the buffer is parked for the next submit
    std::vector<int64_t> buf;
    buf.swap(r.tok);
    buf.clear();
    std::lock_guard<std::mutex> l(c.intake_mu);
    if (c.spare_tok.size() < 256) c.spare_tok.push_back(std::move(buf));
  }
  return rc;
}

int alora_sched_info(void* s, int32_t h, int64_t* out) {
  if (!s || !out || h < 0 || h >= static_cast<int32_t>(C(s)->reqs.size())) return ALORA_EINVAL;
  const Req& r = C(s)->reqs[h];
  out[0] = r.processed;
  out[1] = r.hit;
  out[2] = r.computed;
  out[3] = r.n_gen;
  out[4] = r.state;
  out[5] = static_cast<int64_t>(r.blocks.size());
  out[6] = r.n_reused;
  out[7] = r.failed ? 1 : 0;
  return ALORA_OK;
}

int64_t alora_sched_blocks(void* s, int32_t h, int32_t* out, int64_t cap) {
  if (!s || h < 0 || h >= static_cast<int32_t>(C(s)->reqs.size())) return ALORA_EINVAL;
  const Req& r = C(s)->reqs[h];
  const int64_t n = static_cast<int64_t>(r.blocks.size());
  if (out) std::memcpy(out, r.blocks.data(), static_cast<size_t>(std::min(n, cap)) * sizeof(int32_t));
  return n;
}

int64_t alora_sched_owned_total(void* s) {
  if (!s) return ALORA_EINVAL;
  int64_t t = 0;
  for (const Req& r : C(s)->reqs) t += static_cast<int64_t>(r.blocks.size());
  return t;
}

}  // extern "C"
