// Generates tests/golden/model/ with the REFERENCE's own writers
// (/root/reference/proj/src/bundle.cpp, src/graph.cpp): a tensor bundle with
// the bit patterns the reference tests use (signed zero, subnormal, NaN
// payload, -inf; t/unit/test_bundle.cpp:28-47) and the model_format.md
// example graph with its weights. Build + run: tests/golden/make_model_golden.sh
#include <bit>
#include <cstdint>
#include <filesystem>

#include "widthfold/bundle.hpp"
#include "widthfold/graph.hpp"

using namespace widthfold;

int main(int argc, char** argv) {
  const std::filesystem::path out = argc > 1 ? argv[1] : "tests/golden/model";
  std::filesystem::create_directories(out);
  auto fb = [](std::uint32_t b) { return std::bit_cast<float>(b); };
  TensorBundle b;
  b.add("zeros", DenseTensor::zeros({2, 2}));
  b.add("tricky", DenseTensor({6}, {fb(0x80000000u), fb(0x00000001u), fb(0x7fc00abcu), fb(0xff800000u), 1.5f, -2.25f}));
  std::vector<float> r(60);
  for (int i = 0; i < 60; ++i) r[i] = fb(0x3f800000u + 0x9e3779u * static_cast<std::uint32_t>(i)) - 1.5f;
  b.add("random", DenseTensor({3, 4, 5}, r));
  write_bundle(b, out / "bundle.json");

  // docs/model_format.md example: x(1,32,64,1) -> conv2d(w0: 5x1x1x1) -> bias_add(b0) -> y
  Graph g;
  auto node = [](std::string id, OpKind op, std::vector<std::string> in) {
    Node n;
    n.id = std::move(id);
    n.op = op;
    n.inputs = std::move(in);
    return n;
  };
  Node x = node("x", OpKind::Input, {});
  x.shape = {1, 32, 64, 1};
  Node w = node("w", OpKind::Constant, {});
  w.tensor = "w0";
  Node bb = node("b", OpKind::Constant, {});
  bb.tensor = "b0";
  Node conv = node("conv", OpKind::Conv2d, {"x", "w"});
  Node bias = node("bias", OpKind::BiasAdd, {"conv", "b"});
  Node y = node("y", OpKind::Output, {"bias"});
  g.nodes = {x, w, bb, conv, bias, y};
  g.weights.add("w0", DenseTensor({5, 1, 1, 1}, {0.5f, -1.0f, 2.0f, 0.25f, -0.75f}));
  g.weights.add("b0", DenseTensor({1}, {0.125f}));
  write_graph(g, out / "model.json");
  return 0;
}
