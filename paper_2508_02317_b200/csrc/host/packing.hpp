// Sequence packing: the producer of the step's packed
// varlen input.  Same contract as the reference's pack / padding_ratio /
// StreamingPacker (packing.hpp:14-75, packing.cpp:10-83): first-fit toward a
// target length, FFD sorts by length descending with ties by ascending id,
// samples are never split, an over-length sample is an error naming it.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace opx {

struct PackSample {
  int64_t id = 0, length = 0;
};
struct PackedRow {
  struct Entry {
    int64_t id = 0, offset = 0, length = 0;
  };
  int64_t capacity = 0;
  std::vector<Entry> entries;
  std::vector<int64_t> boundaries;  // starts at 0, ends at used tokens (cu_seqlens)
  int64_t used() const { return boundaries.empty() ? 0 : boundaries.back(); }
};
enum class PackPolicy { first_fit_decreasing = 0, first_fit_arrival = 1 };

struct PackError : std::runtime_error {
  int64_t sample_id;
  PackError(int64_t id, const std::string& w) : std::runtime_error(w), sample_id(id) {}
};

// First fit via a max-tree over the rows' free space: O(n log rows) instead of
// the reference's O(n * rows) scan, same placement (leftmost row that fits).
std::vector<PackedRow> pack(const std::vector<PackSample>& samples, int64_t target, PackPolicy policy);
double padding_ratio(const std::vector<PackedRow>& rows);

class StreamingPacker {
 public:
  StreamingPacker(int64_t target, PackPolicy policy, int64_t buffer_factor = 4)
      : target_(target), policy_(policy), factor_(buffer_factor) {}
  std::vector<PackedRow> push(const PackSample& s);
  std::vector<PackedRow> flush();
  int64_t buffered_tokens() const { return tokens_; }

 private:
  int64_t target_;
  PackPolicy policy_;
  int64_t factor_;
  std::vector<PackSample> buf_;
  int64_t tokens_ = 0;
};

}  // namespace opx
