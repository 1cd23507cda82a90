// B200 mirror of the reference partition API (/root/reference/proj/include/seqpar/partition.hpp).
// Pure host integer code: which global positions each SP group index owns, padding quantum,
// causal pair counts. Same names, argument meaning and ConfigError behaviour.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace seqpar {

// tensor.hpp:18-26 (ShapeError / ConfigError / StateError)
struct ShapeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StateError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

enum class SplitMode { naive, zigzag, usp };  // partition.hpp:14
const char* split_mode_name(SplitMode m);
SplitMode split_mode_from_string(const std::string& s);

// partition.hpp:21-36
struct ShardLayout {
  SplitMode mode = SplitMode::naive;
  int sp = 1;
  int64_t global_len = 0;
  int u_degree = 0;
  int r_degree = 0;
  std::vector<std::vector<int64_t>> owned;

  static ShardLayout make_naive(int64_t len, int sp);    // partition.cpp:37-51
  static ShardLayout make_zigzag(int64_t len, int sp);   // partition.cpp:53-73
  static ShardLayout make_usp(int64_t len, int ulysses_degree, int ring_degree);  // :75-103
  // Extension (not in the reference): the sequence cut into `blocks` equal blocks, each split
  // zigzag over 2*sp chunks (rank i owns chunks i and 2*sp-1-i of every block). blocks = 1 is
  // make_zigzag. Mode stays zigzag (the ring engine's layout); for neat-packed batches whose
  // documents are shorter than the sequence it balances every rank's causal work within each
  // document, which the single zigzag does not (config c5).
  static ShardLayout make_zigzag_blocks(int64_t len, int sp, int blocks);
  int blocks = 1;  // zigzag blocks (1 for every reference layout)

  int64_t local_len() const { return global_len / sp; }
  const std::vector<int64_t>& positions_of(int index) const;
  bool operator==(const ShardLayout& o) const;
};

int64_t causal_pair_count(const ShardLayout& layout, int index);  // partition.cpp:118-122
std::vector<int64_t> make_position_ids(const ShardLayout& layout, int index);  // :160-162
int64_t pad_length(int64_t len, int sp, int64_t cutoff_len, bool pad_to_cutoff = false);  // :179-200
int pick_xtuner_insp(int heads, int sp, int head_dim);  // attention.cpp:354-366

// Closed-form per-rank fwd+bwd bytes in the reference's own accounting (f64 elements, KV
// expanded to q heads): report.cpp:906-941.
int64_t ulysses_bytes(int64_t bs, int64_t len, int64_t heads, int64_t head_dim, int sp);
int64_t ring_bytes(int64_t bs, int64_t len, int64_t heads, int64_t head_dim, int sp);
int64_t dummy_head_bytes(int64_t bs, int64_t len, int64_t heads, int64_t head_dim, int sp);
int64_t xtuner_bytes(int64_t bs, int64_t len, int64_t heads, int64_t head_dim, int sp);
int64_t usp_bytes(int64_t bs, int64_t len, int64_t heads, int64_t head_dim, int u, int r);

// ---- batches, padding and neat-packing metadata (partition.hpp:92-125, partition.cpp:164-227)
constexpr int64_t kIgnoreLabel = -100;
constexpr int64_t kNoImage = -1;
constexpr int64_t kNoSegment = -1;

struct TrainBatch {  // partition.hpp:96-105
  std::vector<int64_t> tokens;
  std::vector<int64_t> labels;        // kIgnoreLabel marks unsupervised slots
  std::vector<int64_t> position_ids;  // [0..len) before sharding
  std::vector<int64_t> segment_ids;   // optional (empty when absent)
  std::vector<int64_t> image_map;     // optional; kNoImage for text positions
  int64_t len() const { return static_cast<int64_t>(tokens.size()); }
  void validate() const;  // partition.cpp:164-177
};

// partition.cpp:202-215: extends every field to pad_length(len, sp, cutoff, pad_to_cutoff)
// with its sentinel (pad_token, kIgnoreLabel, iota positions, kNoSegment, kNoImage).
TrainBatch pad_batch(const TrainBatch& batch, int sp, int64_t pad_token, int64_t cutoff_len,
                     bool pad_to_cutoff = false);
// partition.cpp:217-220 / :124-139: the layout's rows of any per-position int64 field
std::vector<int64_t> shard(const std::vector<int64_t>& values, const ShardLayout& layout, int index);
std::vector<int64_t> split_position_map(const std::vector<int64_t>& image_map,
                                        const ShardLayout& layout, int index);

// B200 bridge from the packed batch to the varlen kernels (the reference keeps segment ids
// but never wires them into attention, model.cpp:339-351): consecutive runs of equal segment
// ids become documents (a kNoSegment tail — pad_batch padding — is one more document, so real
// tokens never attend to padding), and rope position ids restart at 0 in every document.
std::vector<int64_t> documents_from_segments(const std::vector<int64_t>& segment_ids);
std::vector<int64_t> document_position_ids(const std::vector<int64_t>& doc_lens);

// Contiguous position runs of a position list: rows [row0, row0+n) hold positions
// [pos0, pos0+n). The kernels work on runs instead of per-row position arrays.
struct PosRun {
  int64_t row0, pos0, n;
};
std::vector<PosRun> position_runs(const std::vector<int64_t>& positions);

}  // namespace seqpar
