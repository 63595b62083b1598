// Host planner for the shared-prefix paged attention (attn_grp_kernel, attn_bf16.cu).
//
// The reference runs paged_attention once per span (model.py:149-187, looped at model.py:243): every
// request re-reads its whole cached context. With base-aligned block hashing (kv_cache.py:72-96) the
// requests of one conversation evaluated on different adapters hold the SAME physical prefix blocks
// (the eval turn of a multi-adapter pipeline: 8 adapters x one 8k conversation), so their attention
// over that prefix is one computation over one KV stream with 8x the query rows. This planner finds
// those groups from the step's block tables and emits the work list the kernel runs:
//
//   set    = the query rows of a group (or of one ungrouped span), GQA-packed 128 rows per M-tile
//   item   = (set, M-tile, KV partition): one CTA per item and kv head; its segments are streamed in
//            order through one online softmax, so a row's shared-prefix keys and its own private keys
//            (the rest of its sequence, causal) end in one (m, l, O) state
//   seg    = (block-table row, key range [k_lo, k_hi), row filter): the shared prefix of a group is read
//            through its first member's table (identical block ids), a private segment only for the rows
//            of its span (every other row of the tile is masked)
//
// When the items cannot fill the machine, the longest segment of each item of a set is split into KV
// partitions; a partition writes (m, l, O) partials and attn_merge combines them in partition order
// (deterministic). Output blob (int32), all offsets relative to its start:
//   [0] n_items [1] n_segs [2] n_sets [3] max_parts [4] merge_rows [5] unique kv tokens (for the profiler)
//   [6] total key tiles over all items (one kv head) [7] 0
//   items[n_items][8]: set, mtile, seg_begin, seg_end, p_index (-1 = final output), cached_keys, tiles, 0
//   segs[n_segs][4]:   table span, k_lo, k_hi, filter span (-1 = every row)
//   sets[n_sets][2]:   tok_off, n_tok           set_tok[M]: packed token rows           sp_np[S]

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <unordered_map>
#include <vector>

#include "../../include/alora_sm100a.h"

namespace {

// packed query rows per item: the kernel runs MT = 2 tcgen05 query tiles of 128 rows per CTA (ALORA_ATTN_MT=1:
// one; the launcher in attn_bf16.cu reads the same variable)
int item_rows() {
  static const int mt = getenv("ALORA_ATTN_MT") ? std::max(1, std::min(2, atoi(getenv("ALORA_ATTN_MT")))) : 2;
  return 128 * mt;
}
constexpr int kKT = 64;    // keys per KV tile
constexpr int kMaxParts = 8;
constexpr int kNumSMs = 148;

struct Item {
  int set, mtile, seg_begin, seg_end, p_index, cached, tiles;
};

}  // namespace

extern "C" int64_t alora_plan_attention(int32_t S, const int32_t* cu_q, const int32_t* start_pos,
                                        const int32_t* block_table, int32_t max_blocks, int32_t B, int32_t H,
                                        int32_t Hkv, int32_t D, int32_t flags, int64_t partial_cap_bytes,
                                        int32_t* out, int64_t out_cap) {
  if (S < 1 || !cu_q || !start_pos || !block_table || B < 1 || H < 1 || Hkv < 1 || H % Hkv || max_blocks < 1)
    return ALORA_EINVAL;
  const int G = H / Hkv;
  const int M = cu_q[S];
  std::vector<int> end(S), nblk(S);
  for (int s = 0; s < S; ++s) {
    const int n = cu_q[s + 1] - cu_q[s];
    if (n < 1 || start_pos[s] < 0) return ALORA_EINVAL;
    end[s] = start_pos[s] + n;
    nblk[s] = (end[s] + B - 1) / B;
    if (nblk[s] > max_blocks) return ALORA_EINVAL;
  }
  auto tab = [&](int s, int j) { return block_table[(int64_t)s * max_blocks + j]; };

  // 1. groups: spans whose tables start with the same physical blocks, over keys every member has cached
  std::vector<int> group_of(S, -1), shared_keys;
  std::vector<std::vector<int>> groups;
  if (flags & 1) {
    std::unordered_map<int, std::vector<int>> by_first;
    for (int s = 0; s < S; ++s)
      if (start_pos[s] >= 2 * kKT) by_first[tab(s, 0)].push_back(s);
    std::vector<std::vector<int>> cands;
    for (auto& kv : by_first)
      if (kv.second.size() >= 2) cands.push_back(kv.second);
    std::sort(cands.begin(), cands.end(), [](const auto& a, const auto& b) { return a[0] < b[0]; });
    for (auto& mem : cands) {
      int min_start = start_pos[mem[0]];
      for (int s : mem) min_start = std::min(min_start, start_pos[s]);
      int common = min_start / B;  // only blocks wholly before every member's first computed token
      for (size_t i = 1; i < mem.size(); ++i) {
        int j = 0;
        while (j < common && tab(mem[i], j) == tab(mem[0], j)) ++j;
        common = j;
      }
      const int P = (common * B) / kKT * kKT;
      if (P < 2 * kKT) continue;
      for (int s : mem) group_of[s] = (int)groups.size();
      groups.push_back(mem);
      shared_keys.push_back(P);
    }
  }

  // 2. sets (one per group, one per ungrouped span; spans in step order inside a set)
  std::vector<int> set_tok;
  std::vector<int> set_off, set_n, set_group;  // set_group: group id or -(span+1)
  set_tok.reserve(M);
  for (int s = 0; s < S; ++s) {
    if (group_of[s] >= 0) {
      const int g = group_of[s];
      if (groups[g][0] != s) continue;  // emitted with its group's first member
      set_off.push_back((int)set_tok.size());
      for (int m : groups[g])
        for (int r = cu_q[m]; r < cu_q[m + 1]; ++r) set_tok.push_back(r);
      set_n.push_back((int)set_tok.size() - set_off.back());
      set_group.push_back(g);
    } else {
      set_off.push_back((int)set_tok.size());
      for (int r = cu_q[s]; r < cu_q[s + 1]; ++r) set_tok.push_back(r);
      set_n.push_back(cu_q[s + 1] - cu_q[s]);
      set_group.push_back(-(s + 1));
    }
  }
  const int n_sets = (int)set_off.size();
  std::vector<int> row_span(M);
  for (int s = 0; s < S; ++s)
    for (int r = cu_q[s]; r < cu_q[s + 1]; ++r) row_span[r] = s;

  // 3. items (one per set M-tile) and their segments
  std::vector<Item> items;
  std::vector<int> segs;  // 4 per segment
  std::vector<int> item_set_first(n_sets + 1, 0);
  auto add_seg = [&](int table_span, int lo, int hi, int filter) {
    if (hi <= lo) return;
    segs.push_back(table_span);
    segs.push_back(lo);
    segs.push_back(hi);
    segs.push_back(filter);
  };
  auto tiles_of = [&](int b, int e) {
    int t = 0;
    for (int i = b; i < e; ++i) t += (segs[4 * i + 2] - segs[4 * i + 1] + kKT - 1) / kKT;
    return t;
  };
  int64_t unique_kv = 0;
  for (int q = 0; q < n_sets; ++q) {
    item_set_first[q] = (int)items.size();
    const int R = set_n[q] * G;
    const int g = set_group[q];
    const int P = g >= 0 ? shared_keys[g] : 0;
    if (g >= 0) {
      unique_kv += P;
      for (int m : groups[g]) unique_kv += end[m] - P;
    } else {
      unique_kv += end[-g - 1];
    }
    const int QT = item_rows();
    for (int mt = 0; mt * QT < R; ++mt) {
      const int r0 = mt * QT, r1 = std::min(R, r0 + QT) - 1;
      const int t0 = r0 / G, t1 = r1 / G;  // token range of the tile within the set
      Item it{};
      it.set = q;
      it.mtile = mt;
      it.seg_begin = (int)segs.size() / 4;
      it.p_index = -1;
      int cached = 1 << 30;
      if (g >= 0) add_seg(groups[g][0], 0, P, -1);
      // private / causal segment of every span touched by the tile, over its own table
      int tk = t0;
      while (tk <= t1) {
        const int row = set_tok[set_off[q] + tk];
        const int s = row_span[row];
        int last = tk;
        while (last + 1 <= t1 && row_span[set_tok[set_off[q] + last + 1]] == s) ++last;
        const int last_pos = start_pos[s] + (set_tok[set_off[q] + last] - cu_q[s]);
        add_seg(s, P, last_pos + 1, g >= 0 ? s : -1);
        cached = std::min(cached, start_pos[s]);
        tk = last + 1;
      }
      it.seg_end = (int)segs.size() / 4;
      it.cached = (cached / B) * B;
      it.tiles = tiles_of(it.seg_begin, it.seg_end);
      items.push_back(it);
    }
  }
  item_set_first[n_sets] = (int)items.size();

  // 4. KV partitions: pick one split count per set so the item count fills the SMs (1 tcgen05 CTA per SM at
  //    D=128, 2 at D=64) without making CTAs so short that their fixed cost dominates
  const int slots = kNumSMs * ((D == 64 && item_rows() == 128) ? 2 : 1);  // resident CTAs
  const double t_tile = 0.35e-6, t_fix = 5e-6;
  int64_t total_tiles = 0;
  int max_tiles = 0;
  for (auto& it : items) {
    total_tiles += it.tiles;
    max_tiles = std::max(max_tiles, it.tiles);
  }
  const int64_t n_items0 = (int64_t)items.size() * Hkv;
  int best_p = 1;
  double best = 1e30;
  if (!(flags & 2)) {
    for (int p = 1; p <= kMaxParts; ++p) {
      if (p > 1 && max_tiles < 4 * p) break;
      // partial storage for every row of every split set
      const int64_t need = (int64_t)p * M * H * (D + 2) * 4;
      if (p > 1 && need > partial_cap_bytes) break;
      const double waves = std::ceil((double)n_items0 * p / slots);
      const double per = (double)max_tiles / p * t_tile + t_fix;
      const double total = std::max(waves * per, (double)total_tiles * Hkv * t_tile / slots + t_fix);
      if (total < best * 0.97) {
        best = total;
        best_p = p;
      }
    }
    static const int force_p = getenv("ALORA_ATTN_PARTS") ? atoi(getenv("ALORA_ATTN_PARTS")) : 0;  // A/B
    if (force_p > 0) best_p = std::min(force_p, kMaxParts);
  }
  std::vector<Item> final_items;
  std::vector<int> final_segs;
  std::vector<int> sp_np(S, 1);
  int max_np = 1, merge_rows = 0;
  for (int q = 0; q < n_sets; ++q) {
    int set_max = 0;
    for (int i = item_set_first[q]; i < item_set_first[q + 1]; ++i) set_max = std::max(set_max, items[i].tiles);
    const int p = (best_p > 1 && set_max >= 4 * best_p) ? best_p : 1;
    if (p > 1) {
      max_np = std::max(max_np, p);
      const int g = set_group[q];
      if (g >= 0) {
        for (int m : groups[g]) sp_np[m] = p;
      } else {
        sp_np[-g - 1] = p;
      }
      merge_rows += set_n[q];
    }
    for (int i = item_set_first[q]; i < item_set_first[q + 1]; ++i) {
      const Item& it = items[i];
      if (p == 1) {
        Item o = it;
        o.seg_begin = (int)final_segs.size() / 4;
        for (int j = it.seg_begin; j < it.seg_end; ++j) final_segs.insert(final_segs.end(), &segs[4 * j], &segs[4 * j + 4]);
        o.seg_end = (int)final_segs.size() / 4;
        final_items.push_back(o);
        continue;
      }
      // split the first (longest: shared prefix or the span's causal range) segment into p tile-aligned ranges;
      // the last partition also carries the remaining segments
      const int* s0 = &segs[4 * it.seg_begin];
      const int lo = s0[1], hi = s0[2];
      const int ntile = (hi - lo + kKT - 1) / kKT;
      for (int part = 0; part < p; ++part) {
        const int a = lo + (int)((int64_t)ntile * part / p) * kKT;
        const int b = part == p - 1 ? hi : lo + (int)((int64_t)ntile * (part + 1) / p) * kKT;
        Item o = it;
        o.p_index = part;
        o.seg_begin = (int)final_segs.size() / 4;
        if (b > a) final_segs.insert(final_segs.end(), {s0[0], a, b, s0[3]});
        if (part == p - 1)
          for (int j = it.seg_begin + 1; j < it.seg_end; ++j)
            final_segs.insert(final_segs.end(), &segs[4 * j], &segs[4 * j + 4]);
        o.seg_end = (int)final_segs.size() / 4;
        int t = 0;
        for (int j = o.seg_begin; j < o.seg_end; ++j)
          t += (final_segs[4 * j + 2] - final_segs[4 * j + 1] + kKT - 1) / kKT;
        o.tiles = t;
        // an empty partition (short first segment) still writes an empty partial (l = 0) for the merge
        final_items.push_back(o);
      }
    }
  }
  // longest items first: the short private / tail items fill the last wave
  std::stable_sort(final_items.begin(), final_items.end(), [](const Item& x, const Item& y) { return x.tiles > y.tiles; });

  const int n_items = (int)final_items.size(), n_segs = (int)final_segs.size() / 4;
  const int64_t need = 8 + 8LL * n_items + final_segs.size() + 2LL * n_sets + M + S;
  if (!out || out_cap < need) return -need;
  int64_t total = 0;
  for (auto& it : final_items) total += it.tiles;
  out[0] = n_items;
  out[1] = n_segs;
  out[2] = n_sets;
  out[3] = max_np;
  out[4] = merge_rows;
  out[5] = (int32_t)std::min<int64_t>(unique_kv, INT32_MAX);
  out[6] = (int32_t)std::min<int64_t>(total, INT32_MAX);
  out[7] = 0;
  int32_t* p = out + 8;
  for (auto& it : final_items) {
    const int32_t rec[8] = {it.set, it.mtile, it.seg_begin, it.seg_end, it.p_index, it.cached, it.tiles, 0};
    std::memcpy(p, rec, sizeof(rec));
    p += 8;
  }
  std::memcpy(p, final_segs.data(), final_segs.size() * 4);
  p += final_segs.size();
  for (int q = 0; q < n_sets; ++q) {
    *p++ = set_off[q];
    *p++ = set_n[q];
  }
  std::memcpy(p, set_tok.data(), (size_t)M * 4);
  p += M;
  std::memcpy(p, sp_np.data(), (size_t)S * 4);
  p += S;
  return p - out;
}
