// graph.hpp -- the rewrite-rule pass and the interpreter of the reference
// mini-IR, B200-native.
//
// Mirrors /root/reference/proj/include/widthfold/{graph,pass,interpreter}.hpp
// for the conv path: the same Node/Graph/FoldFactor/RewriteReport/PassResult
// names and the same pass contract (total, idempotent, value ids preserved,
// sole-consumer bias_add folded along -- src/pass.cpp:89-218), but
//   * legality is the generalized device fold (KW > 1, stride, padding;
//     SURVEY.md Appendix A) instead of the KW == 1 rule (src/fold.cpp:51-65);
//   * a rewritten conv becomes ONE FoldedConv2d node (the tcgen05 kernel with
//     the bias fused into its epilogue) instead of reshape -> block-diagonal
//     conv -> [bias_add] -> reshape: the reshapes are zero-copy views on the
//     device and the expansion is packed once per weights at execution;
//   * interpret() runs every node on the GPU (ExecMode::Dense/Grouped: the
//     exact-order fp32 conv, src/refconv.cpp:57-78; FoldedConv2d: the folded
//     kernel in TF32 -- the graph values are fp32 like the reference's).
// Out of scope: JSON model files and bundles, the matmul
// branch of the pass; Matmul nodes execute as an exact 1x1 conv.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "widthfold.hpp"

namespace widthfold {

enum class OpKind { Input, Output, Constant, Conv2d, Matmul, BiasAdd, Reshape, FoldedConv2d };
const char* to_string(OpKind kind);
OpKind op_kind_from_string(const std::string& name);

// The reference DenseTensor's role for graph values: f32, row-major, host.
struct HostTensor {
  Shape shape;
  std::vector<float> data;
};

struct Node {
  std::string id;
  OpKind op = OpKind::Input;
  std::vector<std::string> inputs;
  Shape shape;                 // Input: declared shape; Reshape: target shape
  std::string tensor;          // Constant: key into weights
  std::int64_t stride_h = 1;   // Conv2d / FoldedConv2d
  std::int64_t stride_w = 1;
  std::int64_t groups = 1;     // Conv2d: block-diagonal filter with G groups (dense math)
  std::int64_t pad_h = 0;      // extension: symmetric zero padding (reference convs are VALID)
  std::int64_t pad_w = 0;
  std::int64_t factor = 0;     // FoldedConv2d: the device fold factor
  bool bias = false;           // FoldedConv2d: inputs[2] is a bias constant fused in the epilogue
  Dtype dtype = Dtype::TF32;   // FoldedConv2d: tensor-core input dtype (TF32; BF16/F16 cast on the device)
  Shape out_shape;             // filled in by infer_shapes
};

struct Graph {
  std::vector<Node> nodes;
  std::map<std::string, HostTensor> weights;
  const Node* find(const std::string& id) const;
  Node* find(const std::string& id);
  std::vector<std::string> input_ids() const;
  std::vector<std::string> output_ids() const;
};

// ShapeInferenceFailure, MissingInput: widthfold/errors.hpp

// Structural validation plus per-node output shapes (include/widthfold/graph.hpp:48).
Graph infer_shapes(Graph g);
ConvSpec conv_spec_of(const Graph& g, const Node& node);

struct CostEstimate {
  std::uint64_t macs = 0;         // useful MACs (count_macs of every conv / matmul)
  std::uint64_t issued_macs = 0;  // what the device executes (folded convs: tensor-core MACs)
  bool aligned = true;            // every remaining conv's Cin a multiple of `align`
};
CostEstimate cost(const Graph& g, std::int64_t align);

struct FoldFactor {  // include/widthfold/pass.hpp:14-20
  static FoldFactor automatic() { return FoldFactor{}; }
  static FoldFactor fixed(std::int64_t f) { return FoldFactor{f}; }
  bool is_auto() const { return !value.has_value(); }
  std::optional<std::int64_t> value;
};

struct NodeDecision {
  std::string id;
  OpKind kind = OpKind::Conv2d;
  bool applied = false;
  FoldPlan plan;
  std::string note;
};

struct RewriteReport {
  std::vector<NodeDecision> decisions;
  CostEstimate before;
  CostEstimate after;
  std::size_t applied_count() const;
};

struct PassResult {
  Graph graph;
  RewriteReport report;
};

// Rewrites every conv2d the device fold applies to into a FoldedConv2d
// (TF32 tensor cores; a sole-consumer constant bias_add is fused). Never
// fails on legality: skipped nodes carry their FoldReason. Idempotent.
// precision: the folded nodes' tensor-core dtype -- TF32 (default; within
// 1e-3 of the f32 graph) or BF16 / F16 (values cast on the device, 1e-2).
PassResult width_fold_pass(Graph g, FoldFactor factor, std::int64_t align, Dtype precision = Dtype::TF32);

enum class ExecMode { Dense, Grouped, Device };
using TensorMap = std::map<std::string, HostTensor>;

// Executes the graph on the current CUDA device, returns the output values.
TensorMap interpret(const Graph& g, const TensorMap& inputs, ExecMode mode = ExecMode::Device);

}  // namespace widthfold
