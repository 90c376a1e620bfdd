// model_io.hpp -- the model format either side of the device path (SURVEY.md
// 8.F-4, formats only; the CLI stays out of scope): tensor bundles and graph
// JSON files, as specified by /root/reference/proj/docs/model_format.md and
// the reference's bundle.hpp / graph.hpp read/write functions
// (include/widthfold/bundle.hpp:14-39, include/widthfold/graph.hpp:68-70).
//
//   * A bundle is a JSON manifest {"tensors": [{name, shape, dtype, file,
//     byte_offset}]} plus raw little-endian blobs with no header
//     (src/bundle.cpp:83-182). Values move through their bit patterns, so
//     signed zeros, subnormals and NaN payloads round-trip exactly.
//   * dtype: "f32" as in the reference (v1 accepts nothing else,
//     src/bundle.cpp:121-124) plus the device dtypes "bf16" and "f16"
//     (2-byte little-endian), so a model can ship the weights the tensor
//     cores consume.
//   * A graph file is {"nodes": [...], "edges": [{from, to, port}],
//     "weights": manifest path | null} (src/graph.cpp:263-339); node
//     attributes as the reference writes them (shape / tensor / stride +
//     groups), plus this build's extensions: "pad" on conv2d, and the
//     folded_conv2d node of the device pass ("factor", "pad", "bias").
// Errors mirror the reference's: ManifestParse (malformed JSON / fields,
// duplicate names, unknown dtype), BlobSizeMismatch (a tensor that does not
// fit its blob), IoFailure (filesystem).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "graph.hpp"

namespace widthfold {

// ManifestParse, BlobSizeMismatch, IoFailure: widthfold/errors.hpp

// One bundle tensor: shape, dtype tag and the little-endian payload bytes.
struct BundleTensor {
  Shape shape;
  std::string dtype = "f32";      // "f32" | "bf16" | "f16"
  std::vector<std::uint8_t> bytes;
  std::int64_t numel() const;
  std::vector<float> to_f32() const;  // exact (every bf16/f16 value is an f32 value)
  static BundleTensor from_f32(Shape shape, const float* data);
};

int dtype_bytes(const std::string& dtype);  // 4 / 2; throws ManifestParse for anything else

// Named tensors in insertion order (bundle.hpp:14-30).
class TensorBundle {
 public:
  void add(std::string name, BundleTensor t);  // ManifestParse on a duplicate name
  bool contains(const std::string& name) const;
  const BundleTensor& at(const std::string& name) const;  // ManifestParse if absent
  void remove(const std::string& name);
  const std::vector<std::pair<std::string, BundleTensor>>& entries() const { return entries_; }
  std::size_t size() const { return entries_.size(); }

 private:
  std::vector<std::pair<std::string, BundleTensor>> entries_;
};

TensorBundle read_bundle(const std::string& manifest_path);
// Writes the manifest plus one `<stem>.bin` blob beside it.
void write_bundle(const TensorBundle& bundle, const std::string& manifest_path);

// Graph JSON + the bundle it names. Constants of any bundle dtype load as f32
// graph values (the reference graph is f32, graph.hpp:21-45).
Graph read_graph(const std::string& path);
// Writes `path` and, when the graph has constants, `<stem>.weights.json` +
// `<stem>.weights.bin` beside it (f32, src/graph.cpp:315-339).
void write_graph(const Graph& g, const std::string& path);

}  // namespace widthfold
