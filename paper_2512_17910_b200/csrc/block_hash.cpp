// Native block-hash chain: blake2b-128 over the reference's exact byte encoding.
//
// Replaces the per-block Python hashlib loop of
//   /root/reference/pkg/src/aloraserve/kv_cache.py:41-69   (hash_block)
//   kv_cache.py:166-182  (find_cached_prefix chain walk)
//   kv_cache.py:253-260  (commit_and_free re-hash)
// Message per block (all integers little endian):
//   "aloraserve.block.v1" | 0x00            (no parent)
//                         | 0x01 parent[16] (chained)
//   | u32(len(key)) key | u32(block_size) | u32(token) x block_size
// BLAKE2b is RFC 7693 with digest length 16, no key, no salt/personal.

#include <cstdint>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <pthread.h>

#include "../../include/alora_sm100a.h"

namespace {

constexpr uint64_t kIV[8] = {
    0x6a09e667f3bcc908ULL, 0xbb67ae8584caa73bULL, 0x3c6ef372fe94f82bULL, 0xa54ff53a5f1d36f1ULL,
    0x510e527fade682d1ULL, 0x9b05688c2b3e6c1fULL, 0x1f83d9abfb41bd6bULL, 0x5be0cd19137e2179ULL};

constexpr uint8_t kSigma[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},
    {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},
    {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},
    {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},
    {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

inline uint64_t rotr(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

inline uint64_t load64(const uint8_t* p) {
  uint64_t v;
  std::memcpy(&v, p, 8);  // host is little endian (x86_64 / aarch64)
  return v;
}

struct Blake2b {
  uint64_t h[8];
  uint64_t t0 = 0, t1 = 0;
  uint8_t buf[128];
  size_t fill = 0;
  size_t outlen;

  explicit Blake2b(size_t out) : outlen(out) {
    for (int i = 0; i < 8; ++i) h[i] = kIV[i];
    h[0] ^= 0x01010000ULL ^ static_cast<uint64_t>(out);
  }

  void compress(const uint8_t* block, bool last) {
    uint64_t m[16], v[16];
    for (int i = 0; i < 16; ++i) m[i] = load64(block + 8 * i);
    for (int i = 0; i < 8; ++i) {
      v[i] = h[i];
      v[i + 8] = kIV[i];
    }
    v[12] ^= t0;
    v[13] ^= t1;
    if (last) v[14] = ~v[14];
#define G(a, b, c, d, x, y)          \
  do {                               \
    v[a] = v[a] + v[b] + (x);        \
    v[d] = rotr(v[d] ^ v[a], 32);    \
    v[c] = v[c] + v[d];              \
    v[b] = rotr(v[b] ^ v[c], 24);    \
    v[a] = v[a] + v[b] + (y);        \
    v[d] = rotr(v[d] ^ v[a], 16);    \
    v[c] = v[c] + v[d];              \
    v[b] = rotr(v[b] ^ v[c], 63);    \
  } while (0)
#pragma GCC unroll 12
    for (int r = 0; r < 12; ++r) {
      const uint8_t* s = kSigma[r];
      G(0, 4, 8, 12, m[s[0]], m[s[1]]);
      G(1, 5, 9, 13, m[s[2]], m[s[3]]);
      G(2, 6, 10, 14, m[s[4]], m[s[5]]);
      G(3, 7, 11, 15, m[s[6]], m[s[7]]);
      G(0, 5, 10, 15, m[s[8]], m[s[9]]);
      G(1, 6, 11, 12, m[s[10]], m[s[11]]);
      G(2, 7, 8, 13, m[s[12]], m[s[13]]);
      G(3, 4, 9, 14, m[s[14]], m[s[15]]);
    }
#undef G
    for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[i + 8];
  }

  void update(const uint8_t* p, size_t n) {
    while (n > 0) {
      if (fill == 128) {  // only compress a full buffer once more input arrives
        t0 += 128;
        if (t0 < 128) ++t1;
        compress(buf, false);
        fill = 0;
      }
      size_t take = 128 - fill;
      if (take > n) take = n;
      std::memcpy(buf + fill, p, take);
      fill += take;
      p += take;
      n -= take;
    }
  }

  void u32(uint32_t x) {
    uint8_t b[4] = {uint8_t(x), uint8_t(x >> 8), uint8_t(x >> 16), uint8_t(x >> 24)};
    update(b, 4);
  }

  void final(uint8_t* out) {
    t0 += fill;
    if (t0 < fill) ++t1;
    std::memset(buf + fill, 0, 128 - fill);
    compress(buf, true);
    uint8_t full[64];
    std::memcpy(full, h, 64);
    std::memcpy(out, full, outlen);
  }
};

const char kDomain[] = "aloraserve.block.v1";

// Persistent helper threads for the batched hashes: spawning threads inside a process that has torch /
// the CUDA runtime loaded costs ~100 us each (per-thread TLS set-up), more than the hashing they would
// share, so the helpers are created once and parked on a condition variable. run(k, f) runs f on the
// caller plus k-1 helpers; f pulls work from its own atomic counter, so a helper that finds none returns.
class Helpers {
 public:
  void run(int k, const std::function<void()>& f) {
    if (k <= 1) {
      f();
      return;
    }
    std::unique_lock<std::mutex> call(call_mu_);  // one batched call at a time
    {
      std::lock_guard<std::mutex> l(mu_);
      while (static_cast<int>(threads_.size()) < k - 1) {
        threads_.emplace_back([this] { loop(); });
        threads_.back().detach();
      }
      job_ = &f;
      want_ = k - 1;
      pending_ = k - 1;
      ++gen_;
    }
    cv_.notify_all();
    f();
    std::unique_lock<std::mutex> l(mu_);
    done_.wait(l, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void()>* j = nullptr;
      {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return gen_ != seen && want_ > 0; });
        seen = gen_;
        --want_;
        j = job_;
      }
      (*j)();
      std::lock_guard<std::mutex> l(mu_);
      if (--pending_ == 0) done_.notify_all();
    }
  }
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_;
  std::vector<std::thread> threads_;
  const std::function<void()>* job_ = nullptr;
  uint64_t gen_ = 0;
  int want_ = 0, pending_ = 0;
};

// Never destroyed: parked helpers die with the process. A fork()ed child inherits the object but not its
// threads (and perhaps a mutex held by one of them), so the child drops it and lazily builds its own.
std::atomic<Helpers*> g_helpers{nullptr};

void helpers_after_fork_child() { g_helpers.store(nullptr); }

const int g_atfork_registered = pthread_atfork(nullptr, nullptr, helpers_after_fork_child);

Helpers& helpers() {
  Helpers* h = g_helpers.load();
  if (h == nullptr) {
    Helpers* fresh = new Helpers();
    if (g_helpers.compare_exchange_strong(h, fresh)) h = fresh;
    else delete fresh;  // another thread won the race
  }
  return *h;
}

void hash_one(const uint8_t* parent, const uint32_t* tokens, int32_t block_size, const char* key,
              int32_t key_len, uint8_t* out) {
  Blake2b b(16);
  b.update(reinterpret_cast<const uint8_t*>(kDomain), sizeof(kDomain) - 1);
  if (parent == nullptr) {
    uint8_t z = 0;
    b.update(&z, 1);
  } else {
    uint8_t one = 1;
    b.update(&one, 1);
    b.update(parent, 16);
  }
  b.u32(static_cast<uint32_t>(key_len));
  if (key_len > 0) b.update(reinterpret_cast<const uint8_t*>(key), static_cast<size_t>(key_len));
  b.u32(static_cast<uint32_t>(block_size));
  // tokens are already u32 little-endian in memory on the host
  b.update(reinterpret_cast<const uint8_t*>(tokens), static_cast<size_t>(block_size) * 4);
  b.final(out);
}

}  // namespace

extern "C" {

int alora_hash_block(const uint8_t* parent, const uint32_t* tokens, int32_t block_size, const char* key,
                     int32_t key_len, uint8_t* out_digest) {
  if (tokens == nullptr || out_digest == nullptr || block_size < 1 || key_len < 0) return ALORA_EINVAL;
  if (key_len > 0 && key == nullptr) return ALORA_EINVAL;
  hash_one(parent, tokens, block_size, key, key_len, out_digest);
  return ALORA_OK;
}

int alora_hash_chain(const uint8_t* parent, const uint32_t* tokens, int64_t n_blocks, int32_t block_size,
                     const char* key_blob, const int64_t* key_off, uint8_t* out_digests) {
  if (n_blocks < 0 || block_size < 1) return ALORA_EINVAL;
  if (n_blocks == 0) return ALORA_OK;
  if (tokens == nullptr || key_off == nullptr || out_digests == nullptr) return ALORA_EINVAL;
  const uint8_t* prev = parent;
  for (int64_t i = 0; i < n_blocks; ++i) {
    const int64_t k0 = key_off[i], k1 = key_off[i + 1];
    if (k1 < k0) return ALORA_EINVAL;
    hash_one(prev, tokens + i * block_size, block_size, key_blob + k0, static_cast<int32_t>(k1 - k0),
             out_digests + 16 * i);
    prev = out_digests + 16 * i;
  }
  return ALORA_OK;
}

int alora_hash_requests(int32_t n_req, const int64_t* const* tokens, const int64_t* n_blocks, const int64_t* n_base,
                        const char* const* keys, const int32_t* key_lens, int32_t block_size,
                        uint8_t* out_digests, int32_t n_threads) {
  if (n_req < 0 || block_size < 1) return ALORA_EINVAL;
  if (n_req == 0) return ALORA_OK;
  if (tokens == nullptr || n_blocks == nullptr || n_base == nullptr || keys == nullptr || key_lens == nullptr ||
      out_digests == nullptr)
    return ALORA_EINVAL;
  std::vector<int64_t> first(static_cast<size_t>(n_req) + 1, 0);  // digest offset of each request
  for (int32_t r = 0; r < n_req; ++r) {
    if (n_blocks[r] < 0 || key_lens[r] < 0 || (key_lens[r] > 0 && keys[r] == nullptr)) return ALORA_EINVAL;
    first[r + 1] = first[r] + n_blocks[r];
  }
  // Requests admitted together often share their base-key region (several adapters evaluated on one
  // conversation): same n_base and the same tokens there give the same digests, so a follower copies
  // its leader's and hashes only its own tail.
  std::vector<int32_t> leader(static_cast<size_t>(n_req));
  std::vector<int64_t> nbe(static_cast<size_t>(n_req));
  std::vector<uint64_t> fp(static_cast<size_t>(n_req), 0);
  for (int32_t r = 0; r < n_req; ++r) {
    leader[r] = r;
    nbe[r] = n_base[r] < 0 ? 0 : (n_base[r] < n_blocks[r] ? n_base[r] : n_blocks[r]);
    if (nbe[r] == 0) continue;
    const int64_t n = nbe[r] * block_size;
    // a 16-token sample as the fingerprint (a full pass is a serial multiply chain, ~40 us for a
    // 12 x 2k-token batch); memcmp confirms every candidate
    uint64_t h = 0x9e3779b97f4a7c15ULL ^ static_cast<uint64_t>(n);
    for (int k = 0; k < 16; ++k) h = (h ^ static_cast<uint64_t>(tokens[r][(n - 1) * k / 15])) * 0x100000001b3ULL;
    fp[r] = h;
    for (int32_t q = 0; q < r; ++q)
      if (leader[q] == q && nbe[q] == nbe[r] && fp[q] == h &&
          std::memcmp(tokens[q], tokens[r], static_cast<size_t>(n) * sizeof(int64_t)) == 0) {
        leader[r] = q;
        break;
      }
  }
  std::atomic<int> status{ALORA_OK};
  // hash request r's blocks [from, n_blocks) chained from `prev`
  auto hash_tail = [&](int32_t r, int64_t from, const uint8_t* prev, std::vector<uint32_t>& blk) {
    uint8_t* out = out_digests + 16 * first[r];
    for (int64_t i = from; i < n_blocks[r]; ++i) {
      const int64_t* t = tokens[r] + i * block_size;
      for (int32_t j = 0; j < block_size; ++j) {
        if (t[j] < 0 || t[j] > 0xffffffffLL) {
          status.store(ALORA_EINVAL);
          return;
        }
        blk[j] = static_cast<uint32_t>(t[j]);
      }
      // blocks [0, n_base) carry the base key "", the rest the request's key (compute_block_keys)
      const bool base = i < n_base[r];
      hash_one(prev, blk.data(), block_size, base ? "" : keys[r], base ? 0 : key_lens[r], out + 16 * i);
      prev = out + 16 * i;
    }
  };
  auto run = [&](bool followers) {
    int64_t work_blocks = 0;
    std::vector<int32_t> todo;
    for (int32_t r = 0; r < n_req; ++r)
      if ((leader[r] != r) == followers) {
        todo.push_back(r);
        work_blocks += followers ? n_blocks[r] - nbe[r] : n_blocks[r];
      }
    int64_t want = work_blocks / 96;  // a parked helper pays for its wake-up above ~100 blocks
    if (want > n_threads) want = n_threads;
    if (want > static_cast<int64_t>(todo.size())) want = static_cast<int64_t>(todo.size());
    std::atomic<size_t> next{0};
    auto work = [&]() {
      std::vector<uint32_t> blk(static_cast<size_t>(block_size));
      for (size_t k; (k = next.fetch_add(1)) < todo.size();) {
        const int32_t r = todo[k];
        if (!followers) {
          hash_tail(r, 0, nullptr, blk);
        } else {
          uint8_t* out = out_digests + 16 * first[r];
          std::memcpy(out, out_digests + 16 * first[leader[r]], static_cast<size_t>(16 * nbe[r]));
          hash_tail(r, nbe[r], out + 16 * (nbe[r] - 1), blk);
        }
      }
    };
    helpers().run(static_cast<int>(want), work);
  };
  static const bool trace = getenv("ALORA_HASH_TRACE") != nullptr;  // debug: native time of the batch
  const auto t0 = std::chrono::steady_clock::now();
  run(false);
  if (status.load() == ALORA_OK) run(true);
  if (trace) {
    int leaders = 0;
    for (int32_t r = 0; r < n_req; ++r) leaders += leader[r] == r;
    fprintf(stderr, "[hash trace] %d requests (%d leaders), %lld blocks: %.1f us\n", n_req, leaders,
            (long long)first[n_req], std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
  }
  return status.load();
}

int alora_hash_chains(int32_t n_chains, const uint8_t* const* parents, const uint32_t* const* tokens,
                      const int64_t* n_blocks, int32_t block_size, const char* const* key_blobs,
                      const int64_t* const* key_offs, uint8_t* const* out_digests, int32_t n_threads) {
  if (n_chains < 0 || block_size < 1) return ALORA_EINVAL;
  if (n_chains == 0) return ALORA_OK;
  if (tokens == nullptr || n_blocks == nullptr || key_blobs == nullptr || key_offs == nullptr ||
      out_digests == nullptr)
    return ALORA_EINVAL;
  int64_t total = 0;
  for (int32_t c = 0; c < n_chains; ++c) {
    if (n_blocks[c] < 0) return ALORA_EINVAL;
    total += n_blocks[c];
  }
  // chains are independent; each is sequential (block i hashes digest i-1). Threads take whole chains
  // from a shared counter (parked helpers, see Helpers).
  const int64_t kBlocksPerThread = 96;
  int64_t want = total / kBlocksPerThread;
  if (want > n_threads) want = n_threads;
  if (want > n_chains) want = n_chains;
  std::atomic<int32_t> next{0};
  std::atomic<int> status{ALORA_OK};
  auto work = [&]() {
    for (int32_t c; (c = next.fetch_add(1)) < n_chains;) {
      int rc = alora_hash_chain(parents ? parents[c] : nullptr, tokens[c], n_blocks[c], block_size, key_blobs[c],
                                key_offs[c], out_digests[c]);
      if (rc != ALORA_OK) status.store(rc);
    }
  };
  helpers().run(static_cast<int>(want), work);
  return status.load();
}

}  // extern "C"
