// model_io.cpp -- see model_io.hpp. JSON via nlohmann/json (the header-only
// library shipped in the image with cudnn_frontend; the reference uses the
// same library, src/bundle.cpp:9).
#include "model_io.hpp"

#include <cstring>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <map>
#include <set>

#include <nlohmann/json.hpp>

namespace widthfold {

namespace fs = std::filesystem;
using nlohmann::json;

namespace {

std::vector<std::uint8_t> read_file(const fs::path& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoFailure("cannot open " + path.string());
  std::vector<std::uint8_t> bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  if (in.bad()) throw IoFailure("read failed for " + path.string());
  return bytes;
}

json read_json(const fs::path& path) {
  std::ifstream in(path);
  if (!in) throw IoFailure("cannot open " + path.string());
  json j;
  try {
    in >> j;
  } catch (const json::exception& e) {
    throw ManifestParse(path.string() + ": " + e.what());
  }
  return j;
}

void write_text(const fs::path& path, const std::string& text) {
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw IoFailure("cannot write " + path.string());
  out << text << '\n';
  if (!out) throw IoFailure("write failed for " + path.string());
}

std::int64_t shape_numel(const Shape& s) {
  std::int64_t n = 1;
  for (std::int64_t e : s) {
    if (e < 0) throw ManifestParse("negative extent in a tensor shape");
    n *= e;
  }
  return n;
}

// little-endian bit patterns <-> host floats (no arithmetic on the values)
std::uint32_t le32(const std::uint8_t* p) {
  return static_cast<std::uint32_t>(p[0]) | (static_cast<std::uint32_t>(p[1]) << 8) |
         (static_cast<std::uint32_t>(p[2]) << 16) | (static_cast<std::uint32_t>(p[3]) << 24);
}
float f16_to_f32(std::uint16_t h) {  // IEEE binary16 -> binary32, exact (payload bits kept for NaN)
  const std::uint32_t sign = static_cast<std::uint32_t>(h & 0x8000u) << 16;
  const std::uint32_t exp = (h >> 10) & 0x1Fu, man = h & 0x3FFu;
  std::uint32_t bits;
  if (exp == 0x1Fu) {
    bits = sign | 0x7F800000u | (man << 13);
  } else if (exp != 0) {
    bits = sign | ((exp + 112u) << 23) | (man << 13);
  } else if (man == 0) {
    bits = sign;
  } else {  // subnormal half: normalise
    int e = -1;
    std::uint32_t m = man;
    do { m <<= 1; ++e; } while (!(m & 0x400u));
    bits = sign | ((112u - static_cast<std::uint32_t>(e)) << 23) | ((m & 0x3FFu) << 13);
  }
  float f;
  std::memcpy(&f, &bits, 4);
  return f;
}

}  // namespace

int dtype_bytes(const std::string& dtype) {
  if (dtype == "f32") return 4;
  if (dtype == "bf16" || dtype == "f16") return 2;
  throw ManifestParse("unsupported dtype '" + dtype + "' (f32, bf16, f16)");
}

std::int64_t BundleTensor::numel() const { return shape_numel(shape); }

std::vector<float> BundleTensor::to_f32() const {
  const std::int64_t n = numel();
  std::vector<float> out(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) {
    std::uint32_t bits;
    if (dtype == "f32") {
      bits = le32(&bytes[4 * i]);
      std::memcpy(&out[i], &bits, 4);
    } else {
      const std::uint16_t h = static_cast<std::uint16_t>(bytes[2 * i] | (bytes[2 * i + 1] << 8));
      if (dtype == "bf16") {
        bits = static_cast<std::uint32_t>(h) << 16;
        std::memcpy(&out[i], &bits, 4);
      } else {
        out[i] = f16_to_f32(h);
      }
    }
  }
  return out;
}

BundleTensor BundleTensor::from_f32(Shape shape, const float* data) {
  BundleTensor t;
  t.shape = std::move(shape);
  t.dtype = "f32";
  const std::int64_t n = t.numel();
  t.bytes.resize(static_cast<std::size_t>(4 * n));
  for (std::int64_t i = 0; i < n; ++i) {
    std::uint32_t bits;
    std::memcpy(&bits, &data[i], 4);
    for (int k = 0; k < 4; ++k) t.bytes[4 * i + k] = static_cast<std::uint8_t>((bits >> (8 * k)) & 0xFFu);
  }
  return t;
}

void TensorBundle::add(std::string name, BundleTensor t) {
  if (contains(name)) throw ManifestParse("duplicate tensor name '" + name + "' in bundle");
  entries_.emplace_back(std::move(name), std::move(t));
}

bool TensorBundle::contains(const std::string& name) const {
  for (const auto& e : entries_)
    if (e.first == name) return true;
  return false;
}

const BundleTensor& TensorBundle::at(const std::string& name) const {
  for (const auto& e : entries_)
    if (e.first == name) return e.second;
  throw ManifestParse("bundle has no tensor named '" + name + "'");
}

void TensorBundle::remove(const std::string& name) {
  for (auto it = entries_.begin(); it != entries_.end(); ++it)
    if (it->first == name) {
      entries_.erase(it);
      return;
    }
}

TensorBundle read_bundle(const std::string& manifest_path) {
  const fs::path mpath(manifest_path);
  const json m = read_json(mpath);
  if (!m.is_object() || !m.contains("tensors") || !m["tensors"].is_array())
    throw ManifestParse(manifest_path + ": expected an object with a 'tensors' array");
  std::map<std::string, std::vector<std::uint8_t>> blobs;  // file -> bytes, each read once
  TensorBundle bundle;
  for (const auto& e : m["tensors"]) {
    std::string name, file, dtype;
    Shape shape;
    std::uint64_t off = 0;
    try {
      name = e.at("name").get<std::string>();
      file = e.at("file").get<std::string>();
      dtype = e.at("dtype").get<std::string>();
      shape = e.at("shape").get<Shape>();
      off = e.value("byte_offset", std::uint64_t{0});
    } catch (const json::exception& ex) {
      throw ManifestParse(manifest_path + ": bad tensor entry: " + ex.what());
    }
    const int eb = dtype_bytes(dtype);
    auto it = blobs.find(file);
    if (it == blobs.end()) it = blobs.emplace(file, read_file(mpath.parent_path() / file)).first;
    const std::uint64_t want = static_cast<std::uint64_t>(shape_numel(shape)) * static_cast<std::uint64_t>(eb);
    if (off + want > it->second.size())
      throw BlobSizeMismatch("tensor '" + name + "' wants bytes [" + std::to_string(off) + ", " +
                             std::to_string(off + want) + ") but blob '" + file + "' has " +
                             std::to_string(it->second.size()) + " bytes");
    BundleTensor t;
    t.shape = std::move(shape);
    t.dtype = dtype;
    t.bytes.assign(it->second.begin() + static_cast<std::ptrdiff_t>(off),
                   it->second.begin() + static_cast<std::ptrdiff_t>(off + want));
    bundle.add(std::move(name), std::move(t));
  }
  return bundle;
}

void write_bundle(const TensorBundle& bundle, const std::string& manifest_path) {
  const fs::path mpath(manifest_path);
  const std::string blob_name = mpath.stem().string() + ".bin";
  json tensors = json::array();
  std::vector<std::uint8_t> blob;
  for (const auto& [name, t] : bundle.entries()) {
    const std::uint64_t want = static_cast<std::uint64_t>(t.numel()) * static_cast<std::uint64_t>(dtype_bytes(t.dtype));
    if (t.bytes.size() != want) throw BlobSizeMismatch("tensor '" + name + "' payload does not match its shape");
    tensors.push_back({{"name", name}, {"shape", t.shape}, {"dtype", t.dtype}, {"file", blob_name},
                       {"byte_offset", static_cast<std::uint64_t>(blob.size())}});
    blob.insert(blob.end(), t.bytes.begin(), t.bytes.end());
  }
  std::error_code ec;
  if (!mpath.parent_path().empty()) fs::create_directories(mpath.parent_path(), ec);
  {
    std::ofstream out(mpath.parent_path() / blob_name, std::ios::binary | std::ios::trunc);
    if (!out) throw IoFailure("cannot write " + (mpath.parent_path() / blob_name).string());
    out.write(reinterpret_cast<const char*>(blob.data()), static_cast<std::streamsize>(blob.size()));
    if (!out) throw IoFailure("write failed for " + blob_name);
  }
  write_text(mpath, json{{"tensors", tensors}}.dump(2));
}

namespace {

json node_to_json(const Node& n) {
  json j{{"id", n.id}, {"op", to_string(n.op)}};
  switch (n.op) {
    case OpKind::Input:
    case OpKind::Reshape:
      j["shape"] = n.shape;
      break;
    case OpKind::Constant:
      j["tensor"] = n.tensor;
      break;
    case OpKind::Conv2d:
      j["stride"] = {n.stride_h, n.stride_w};
      j["groups"] = n.groups;
      if (n.pad_h || n.pad_w) {
        // extension (reference convs are VALID): a padded conv is written as
        // its own op kind, which the reference reader rejects as unknown
        // (src/graph.cpp:28-32) instead of silently loading it unpadded
        j["op"] = "conv2d_padded";
        j["pad"] = {n.pad_h, n.pad_w};
      }
      break;
    case OpKind::FoldedConv2d:
      j["stride"] = {n.stride_h, n.stride_w};
      j["pad"] = {n.pad_h, n.pad_w};
      j["factor"] = n.factor;
      j["bias"] = n.bias;
      j["dtype"] = n.dtype == Dtype::BF16 ? "bf16" : (n.dtype == Dtype::F16 ? "f16" : "tf32");
      break;
    default:
      break;
  }
  return j;
}

std::pair<std::int64_t, std::int64_t> pair_of(const json& j, const char* key, std::int64_t dflt) {
  const auto v = j.value(key, std::vector<std::int64_t>{dflt, dflt});
  if (v.size() != 2) throw ManifestParse(std::string("'") + key + "' wants 2 entries");
  return {v[0], v[1]};
}

Node node_from_json(const json& j) {
  Node n;
  n.id = j.at("id").get<std::string>();
  try {
    const std::string op = j.at("op").get<std::string>();
    n.op = (op == "conv2d_padded") ? OpKind::Conv2d : op_kind_from_string(op);
  } catch (const std::invalid_argument& e) {
    throw ManifestParse(e.what());  // unknown ops are rejected, not guessed (docs/model_format.md)
  }
  switch (n.op) {
    case OpKind::Input:
    case OpKind::Reshape:
      n.shape = j.at("shape").get<Shape>();
      break;
    case OpKind::Constant:
      n.tensor = j.at("tensor").get<std::string>();
      break;
    case OpKind::Conv2d:
    case OpKind::FoldedConv2d:
      std::tie(n.stride_h, n.stride_w) = pair_of(j, "stride", 1);
      std::tie(n.pad_h, n.pad_w) = pair_of(j, "pad", 0);
      n.groups = j.value("groups", std::int64_t{1});
      if (n.op == OpKind::FoldedConv2d) {
        n.factor = j.at("factor").get<std::int64_t>();
        n.bias = j.value("bias", false);
        const std::string dt = j.value("dtype", std::string("tf32"));
        if (dt == "bf16") n.dtype = Dtype::BF16;
        else if (dt == "f16") n.dtype = Dtype::F16;
        else if (dt == "tf32") n.dtype = Dtype::TF32;
        else throw ManifestParse("folded_conv2d '" + n.id + "': unknown dtype '" + dt + "'");
      }
      break;
    default:
      break;
  }
  return n;
}

}  // namespace

Graph read_graph(const std::string& path) {
  const fs::path gpath(path);
  const json j = read_json(gpath);
  Graph g;
  try {
    if (!j.is_object()) throw ManifestParse(path + ": graph file must be a JSON object");
    for (const auto& jn : j.at("nodes")) g.nodes.push_back(node_from_json(jn));
    std::set<std::string> ids;
    for (const auto& n : g.nodes)
      if (!ids.insert(n.id).second) throw ManifestParse(path + ": duplicate node id '" + n.id + "'");
    // value of `from` becomes input `port` of `to`; ports must be 0..n-1
    std::map<std::string, std::map<std::int64_t, std::string>> wiring;
    for (const auto& je : j.at("edges")) {
      const auto from = je.at("from").get<std::string>();
      const auto to = je.at("to").get<std::string>();
      if (!ids.count(from) || !ids.count(to))
        throw ManifestParse("edge " + from + " -> " + to + " references an unknown node");
      const std::int64_t port = je.value("port", std::int64_t{0});
      if (!wiring[to].emplace(port, from).second)
        throw ManifestParse("node '" + to + "': port " + std::to_string(port) + " wired twice");
    }
    for (auto& n : g.nodes) {
      auto it = wiring.find(n.id);
      if (it == wiring.end()) continue;
      std::int64_t expect = 0;
      for (const auto& [port, from] : it->second) {
        if (port != expect++) throw ManifestParse("node '" + n.id + "': input ports must be 0..n-1");
        n.inputs.push_back(from);
      }
    }
    if (j.contains("weights") && !j.at("weights").is_null()) {
      const TensorBundle b = read_bundle((gpath.parent_path() / j.at("weights").get<std::string>()).string());
      for (const auto& [name, t] : b.entries()) g.weights[name] = HostTensor{t.shape, t.to_f32()};
    }
  } catch (const json::exception& e) {
    throw ManifestParse(path + ": " + e.what());
  }
  return g;
}

void write_graph(const Graph& g, const std::string& path) {
  const fs::path gpath(path);
  json nodes = json::array(), edges = json::array();
  for (const auto& n : g.nodes) {
    nodes.push_back(node_to_json(n));
    for (std::size_t port = 0; port < n.inputs.size(); ++port)
      edges.push_back({{"from", n.inputs[port]}, {"to", n.id}, {"port", static_cast<std::int64_t>(port)}});
  }
  json j{{"nodes", nodes}, {"edges", edges}};
  if (!g.weights.empty()) {
    const std::string wname = gpath.stem().string() + ".weights.json";
    TensorBundle b;
    for (const auto& [name, t] : g.weights) b.add(name, BundleTensor::from_f32(t.shape, t.data.data()));
    write_bundle(b, (gpath.parent_path() / wname).string());
    j["weights"] = wname;
  } else {
    j["weights"] = nullptr;
  }
  write_text(gpath, j.dump(2));
}

}  // namespace widthfold
