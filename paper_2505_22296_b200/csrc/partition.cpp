// Host integer side of the SP layer: layouts, padding, xtuner factor, byte models.
// Semantics follow /root/reference/proj/src/partition.cpp and report.cpp (cited per function);
// the implementation is ours (run-based, no per-element work on the hot path).
#include <algorithm>
#include <numeric>

#include "seqpar/partition.hpp"

namespace seqpar {

const char* split_mode_name(SplitMode m) {
  return m == SplitMode::naive ? "naive" : m == SplitMode::zigzag ? "zigzag" : "usp";
}

SplitMode split_mode_from_string(const std::string& s) {  // partition.cpp:21-26
  if (s == "naive") return SplitMode::naive;
  if (s == "zigzag") return SplitMode::zigzag;
  if (s == "usp") return SplitMode::usp;
  throw ConfigError("unknown split mode '" + s + "'");
}

namespace {
void require_split(int64_t len, int64_t parts, const char* what, int sp) {  // partition.cpp:28-35
  if (sp <= 0) throw ConfigError("sp must be positive");
  if (len <= 0) throw ConfigError("sequence length must be positive");
  if (len % parts) {
    throw ConfigError(std::string(what) + ": length " + std::to_string(len) +
                      (parts == sp ? " not divisible by sp " + std::to_string(sp)
                                   : " not divisible by 2*sp = " + std::to_string(parts)));
  }
}

std::vector<int64_t> span_of(int64_t begin, int64_t n) {
  std::vector<int64_t> v(static_cast<size_t>(n));
  std::iota(v.begin(), v.end(), begin);
  return v;
}
}  // namespace

ShardLayout ShardLayout::make_naive(int64_t len, int sp) {
  require_split(len, sp, "naive split", sp);
  ShardLayout L;
  L.mode = SplitMode::naive;
  L.sp = sp;
  L.global_len = len;
  const int64_t n = len / sp;
  for (int i = 0; i < sp; ++i) L.owned.push_back(span_of(i * n, n));
  return L;
}

ShardLayout ShardLayout::make_zigzag(int64_t len, int sp) {
  require_split(len, sp, "zigzag split", sp);
  require_split(len, 2 * static_cast<int64_t>(sp), "zigzag split", sp);
  ShardLayout L;
  L.mode = SplitMode::zigzag;
  L.sp = sp;
  L.global_len = len;
  const int64_t c = len / (2 * sp);
  for (int i = 0; i < sp; ++i) {
    auto lo = span_of(i * c, c), hi = span_of((2 * sp - 1 - i) * c, c);
    lo.insert(lo.end(), hi.begin(), hi.end());
    L.owned.push_back(std::move(lo));
  }
  return L;
}

ShardLayout ShardLayout::make_zigzag_blocks(int64_t len, int sp, int blocks) {
  if (blocks <= 0) throw ConfigError("zigzag blocks: block count must be positive");
  if (blocks == 1) return make_zigzag(len, sp);
  require_split(len, sp, "zigzag split", sp);
  const int64_t parts = 2 * static_cast<int64_t>(sp) * blocks;
  if (len % parts) {
    throw ConfigError("zigzag blocks: length " + std::to_string(len) + " not divisible by 2*sp*blocks = " +
                      std::to_string(parts));
  }
  ShardLayout L;
  L.mode = SplitMode::zigzag;
  L.sp = sp;
  L.global_len = len;
  L.blocks = blocks;
  const int64_t c = len / parts, bl = len / blocks;
  L.owned.resize(static_cast<size_t>(sp));
  for (int i = 0; i < sp; ++i)
    for (int b = 0; b < blocks; ++b)
      for (int64_t ch : {static_cast<int64_t>(i), 2 * static_cast<int64_t>(sp) - 1 - i}) {
        auto run = span_of(b * bl + ch * c, c);
        L.owned[static_cast<size_t>(i)].insert(L.owned[static_cast<size_t>(i)].end(), run.begin(), run.end());
      }
  return L;
}

ShardLayout ShardLayout::make_usp(int64_t len, int u, int r) {
  if (u <= 0 || r <= 0) throw ConfigError("usp split: degrees must be positive");
  const ShardLayout ring = make_zigzag(len, r);
  const int64_t block = len / r;
  if (block % u) {
    throw ConfigError("usp split: ring block " + std::to_string(block) +
                      " not divisible by ulysses degree " + std::to_string(u));
  }
  ShardLayout L;
  L.mode = SplitMode::usp;
  L.sp = u * r;
  L.global_len = len;
  L.u_degree = u;
  L.r_degree = r;
  const int64_t n = block / u;
  for (int rho = 0; rho < r; ++rho)
    for (int iota = 0; iota < u; ++iota) {
      const auto& b = ring.owned[static_cast<size_t>(rho)];
      L.owned.emplace_back(b.begin() + iota * n, b.begin() + (iota + 1) * n);
    }
  return L;
}

const std::vector<int64_t>& ShardLayout::positions_of(int index) const {
  if (index < 0 || index >= sp) {
    throw ConfigError("layout index " + std::to_string(index) + " out of range for sp " +
                      std::to_string(sp));
  }
  return owned[static_cast<size_t>(index)];
}

bool ShardLayout::operator==(const ShardLayout& o) const {
  return mode == o.mode && sp == o.sp && global_len == o.global_len && blocks == o.blocks && owned == o.owned;
}

int64_t causal_pair_count(const ShardLayout& layout, int index) {
  const auto& p = layout.positions_of(index);
  return std::accumulate(p.begin(), p.end(), int64_t{0}) + static_cast<int64_t>(p.size());
}

std::vector<int64_t> make_position_ids(const ShardLayout& layout, int index) {
  return layout.positions_of(index);
}

int64_t pad_length(int64_t len, int sp, int64_t cutoff_len, bool pad_to_cutoff) {
  if (len <= 0) throw ConfigError("pad_length: length must be positive");
  if (sp <= 0) throw ConfigError("pad_length: sp must be positive");
  const int64_t q = 8 * static_cast<int64_t>(sp);  // PAPER.md:67 (multiple of 8*sp)
  if (pad_to_cutoff) {
    if (cutoff_len % q) {
      throw ConfigError("cutoff_len " + std::to_string(cutoff_len) +
                        " is not a multiple of 8*sp = " + std::to_string(q));
    }
    if (len > cutoff_len) {
      throw ConfigError("sequence of length " + std::to_string(len) + " exceeds cutoff_len " +
                        std::to_string(cutoff_len));
    }
    return cutoff_len;
  }
  const int64_t padded = (len + q - 1) / q * q;
  if (padded > cutoff_len) {
    throw ConfigError("padded length " + std::to_string(padded) + " exceeds cutoff_len " +
                      std::to_string(cutoff_len));
  }
  return padded;
}

int pick_xtuner_insp(int heads, int sp, int head_dim) {
  if (heads <= 0 || sp <= 0 || head_dim <= 0) {
    throw ConfigError("xtuner: heads, sp, and head_dim must be positive");
  }
  const int step = sp / std::gcd(heads, sp);
  for (int f = step; f <= head_dim; f += step)
    if (head_dim % f == 0 && sp % f == 0) return f;
  throw ConfigError("xtuner: no virtual-head factor for heads=" + std::to_string(heads) +
                    ", sp=" + std::to_string(sp) + ", head_dim=" + std::to_string(head_dim));
}

// ---- reference byte accounting (report.cpp:906-941): f64 payloads, KV expanded
namespace {
int64_t local_f64(int64_t bs, int64_t len, int64_t heads, int64_t d, int sp) {
  return bs * (len / sp) * heads * d * 8;
}
}  // namespace

int64_t ulysses_bytes(int64_t bs, int64_t len, int64_t heads, int64_t d, int sp) {
  return 8 * (local_f64(bs, len, heads, d, sp) * (sp - 1) / sp);
}
int64_t ring_bytes(int64_t bs, int64_t len, int64_t heads, int64_t d, int sp) {
  return (6 * static_cast<int64_t>(sp) - 2) * local_f64(bs, len, heads, d, sp);
}
int64_t dummy_head_bytes(int64_t bs, int64_t len, int64_t heads, int64_t d, int sp) {
  return ulysses_bytes(bs, len, (heads + sp - 1) / sp * sp, d, sp);
}
int64_t xtuner_bytes(int64_t bs, int64_t len, int64_t heads, int64_t d, int sp) {
  const int f = pick_xtuner_insp(static_cast<int>(heads), sp, static_cast<int>(d));
  return ulysses_bytes(bs, len, heads, d, sp) + 6 * local_f64(bs, len, heads, d, sp) * (f - 1);
}
int64_t usp_bytes(int64_t bs, int64_t len, int64_t heads, int64_t d, int u, int r) {
  const int64_t hp = u > 1 ? (heads + u - 1) / u * u : heads;
  const int64_t x = local_f64(bs, len, hp, d, u * r);
  int64_t total = 0;
  if (u > 1) total += 8 * (x * (u - 1) / u);
  if (r > 1) total += (6 * static_cast<int64_t>(r) - 2) * x;
  return total;
}

std::vector<PosRun> position_runs(const std::vector<int64_t>& p) {
  std::vector<PosRun> runs;
  for (size_t i = 0; i < p.size(); ++i) {
    if (!runs.empty() && runs.back().pos0 + runs.back().n == p[i] &&
        runs.back().row0 + runs.back().n == static_cast<int64_t>(i)) {
      ++runs.back().n;
    } else {
      runs.push_back({static_cast<int64_t>(i), p[i], 1});
    }
  }
  return runs;
}

// ------------------------------------------------------------------ batches and packing
void TrainBatch::validate() const {
  const size_t n = tokens.size();
  if (n == 0) throw ConfigError("batch has no tokens");
  if (labels.size() != n) throw ConfigError("batch labels length does not match tokens");
  if (position_ids.size() != n) throw ConfigError("batch position_ids length does not match tokens");
  if (!segment_ids.empty() && segment_ids.size() != n)
    throw ConfigError("batch segment_ids length does not match tokens");
  if (!image_map.empty() && image_map.size() != n)
    throw ConfigError("batch image_map length does not match tokens");
}

TrainBatch pad_batch(const TrainBatch& batch, int sp, int64_t pad_token, int64_t cutoff_len,
                     bool pad_to_cutoff) {
  batch.validate();
  const int64_t target = pad_length(batch.len(), sp, cutoff_len, pad_to_cutoff);
  const size_t t = static_cast<size_t>(target);
  TrainBatch out = batch;
  out.tokens.resize(t, pad_token);
  out.labels.resize(t, kIgnoreLabel);
  out.position_ids.resize(t);
  for (size_t i = 0; i < t; ++i) out.position_ids[i] = static_cast<int64_t>(i);
  if (!out.segment_ids.empty()) out.segment_ids.resize(t, kNoSegment);
  if (!out.image_map.empty()) out.image_map.resize(t, kNoImage);
  return out;
}

std::vector<int64_t> shard(const std::vector<int64_t>& values, const ShardLayout& layout, int index) {
  if (static_cast<int64_t>(values.size()) != layout.global_len)
    throw ShapeError("shard: " + std::to_string(values.size()) + " values for a layout of " +
                     std::to_string(layout.global_len));
  std::vector<int64_t> out;
  for (int64_t p : layout.positions_of(index)) out.push_back(values[static_cast<size_t>(p)]);
  return out;
}

std::vector<int64_t> split_position_map(const std::vector<int64_t>& image_map,
                                        const ShardLayout& layout, int index) {
  return shard(image_map, layout, index);
}

std::vector<int64_t> documents_from_segments(const std::vector<int64_t>& seg) {
  std::vector<int64_t> docs, seen;
  for (size_t i = 0; i < seg.size();) {
    size_t j = i + 1;
    while (j < seg.size() && seg[j] == seg[i]) ++j;
    if (seg[i] != kNoSegment) {
      if (std::find(seen.begin(), seen.end(), seg[i]) != seen.end())
        throw ConfigError("segment id " + std::to_string(seg[i]) +
                          " is not one contiguous run; a packed document must be contiguous");
      seen.push_back(seg[i]);
    }
    docs.push_back(static_cast<int64_t>(j - i));
    i = j;
  }
  return docs;
}

std::vector<int64_t> document_position_ids(const std::vector<int64_t>& doc_lens) {
  std::vector<int64_t> ids;
  for (int64_t n : doc_lens) {
    if (n <= 0) throw ConfigError("documents: lengths must be positive");
    for (int64_t i = 0; i < n; ++i) ids.push_back(i);
  }
  return ids;
}

}  // namespace seqpar
