// bindings.cpp -- pybind11 module `paper_2601_11608_b200._core`.
//
// Mirrors the reference binding (/root/reference/proj/python/bindings.cpp:48-207):
// same function names, keyword arguments, plan_dict keys and exception types
// (ShapeMismatchError / IllegalFoldError / DegenerateOutputError are ValueError
// subclasses, bindings.cpp:51-56). Device data crosses as integer pointers plus
// shapes and a cudaStream_t; the Python layer (api.py) maps torch/numpy onto it.
// The GIL is released around every device call.
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cstdint>

#include <pybind11/numpy.h>

#include "graph.hpp"
#include "model_io.hpp"
#include "widthfold.hpp"

namespace py = pybind11;
namespace wf = widthfold;

namespace {

void* P(std::uintptr_t v) { return reinterpret_cast<void*>(v); }
const float* F(std::uintptr_t v) { return reinterpret_cast<const float*>(v); }

wf::Dtype dtype_of(const std::string& s) {
  if (s == "bf16") return wf::Dtype::BF16;
  if (s == "f16" || s == "fp16") return wf::Dtype::F16;
  if (s == "tf32") return wf::Dtype::TF32;
  if (s == "f32" || s == "fp32") return wf::Dtype::F32;
  throw std::invalid_argument("unknown dtype '" + s + "'");
}

py::dict plan_dict(const wf::FoldPlan& plan) {
  py::dict d;
  d["status"] = plan.ok() ? "apply" : "fallback";
  d["reason"] = wf::to_string(plan.reason);
  d["factor"] = plan.factor;
  d["folded_input_shape"] = plan.folded_input_shape;
  d["expanded_filter_shape"] = plan.expanded_filter_shape;
  return d;
}

py::dict raw_dict(const wf_fold_plan& p) {
  py::dict d;
  d["f"] = p.f; d["r"] = p.r; d["c0"] = p.c0; d["kw_f"] = p.kw_f; d["k_f"] = p.k_f; d["cout_f"] = p.cout_f;
  d["oh"] = p.oh; d["ow"] = p.ow; d["wf"] = p.wf; d["wfo"] = p.wfo; d["units_per_px"] = p.units_per_px;
  d["group_size"] = p.group_size; d["n_groups"] = p.n_groups; d["n_tiles"] = p.n_tiles;
  d["tile_rows"] = p.tile_rows; d["wbox"] = p.wbox; d["nrows"] = p.nrows; d["mma_entries"] = p.mma_entries;
  d["packed_bytes"] = p.packed_bytes; d["epi_chunk"] = p.epi_chunk;
  d["variant"] = p.variant == WF_VARIANT_UNFOLDED ? "unfolded" : "fold";
  d["producer"] = p.producer == 0   ? "tma"
                  : p.producer == 1 ? "row-ring"
                  : p.producer == 2 ? "im2col"
                  : p.producer == 3 ? "repitch+tma"
                  : p.producer == 5 ? "ring+tma"
                  : p.producer == 6 ? "gather-direct"
                                    : "gather";
  d["pitched_w"] = p.pitched_w; d["workspace_bytes"] = p.workspace_bytes; d["cta_pair"] = p.cta_pair; d["stage_tiles"] = p.stage_tiles; d["kstep_mode"] = p.kstep_mode;
  d["in_dtype"] = p.in_dtype; d["launch_opts"] = p.launch_opts; d["useful_macs"] = p.useful_macs; d["issued_macs"] = p.issued_macs;
  return d;
}

wf::ConvSpec spec_of(const wf::Shape& in, const wf::Shape& filt, std::int64_t sh, std::int64_t sw, std::int64_t ph,
                     std::int64_t pw) {
  return wf::ConvSpec{in, filt, sh, sw, ph, pw};
}

// ---- graph <-> Python (list of node dicts, dict of float32 arrays) ----------------
using F32Array = py::array_t<float, py::array::c_style | py::array::forcecast>;

wf::HostTensor host_tensor(const F32Array& a) {
  wf::HostTensor t;
  for (py::ssize_t i = 0; i < a.ndim(); ++i) t.shape.push_back(a.shape(i));
  t.data.assign(a.data(), a.data() + a.size());
  return t;
}

F32Array to_array(const wf::HostTensor& t) {
  std::vector<py::ssize_t> shape(t.shape.begin(), t.shape.end());
  F32Array a(shape);
  std::copy(t.data.begin(), t.data.end(), a.mutable_data());
  return a;
}

template <typename T>
T get_or(const py::dict& d, const char* k, T dflt) {
  return d.contains(k) ? d[k].cast<T>() : dflt;
}

wf::Graph graph_of(const py::list& nodes, const py::dict& weights) {
  wf::Graph g;
  for (auto item : weights) g.weights[item.first.cast<std::string>()] = host_tensor(item.second.cast<F32Array>());
  for (auto h : nodes) {
    const py::dict d = h.cast<py::dict>();
    wf::Node n;
    n.id = d["id"].cast<std::string>();
    n.op = wf::op_kind_from_string(d["op"].cast<std::string>());
    n.inputs = get_or<std::vector<std::string>>(d, "inputs", {});
    n.shape = get_or<wf::Shape>(d, "shape", {});
    n.tensor = get_or<std::string>(d, "tensor", "");
    n.stride_h = get_or<std::int64_t>(d, "stride_h", 1);
    n.stride_w = get_or<std::int64_t>(d, "stride_w", 1);
    n.groups = get_or<std::int64_t>(d, "groups", 1);
    n.pad_h = get_or<std::int64_t>(d, "pad_h", 0);
    n.pad_w = get_or<std::int64_t>(d, "pad_w", 0);
    n.factor = get_or<std::int64_t>(d, "factor", 0);
    n.bias = get_or<bool>(d, "bias", false);
    n.dtype = dtype_of(get_or<std::string>(d, "dtype", "tf32"));
    g.nodes.push_back(std::move(n));
  }
  return g;
}

py::list nodes_of(const wf::Graph& g) {
  py::list out;
  for (const auto& n : g.nodes) {
    py::dict d;
    d["id"] = n.id;
    d["op"] = wf::to_string(n.op);
    d["inputs"] = n.inputs;
    if (!n.shape.empty()) d["shape"] = n.shape;
    if (!n.tensor.empty()) d["tensor"] = n.tensor;
    if (n.op == wf::OpKind::Conv2d || n.op == wf::OpKind::FoldedConv2d) {
      d["stride_h"] = n.stride_h;
      d["stride_w"] = n.stride_w;
      d["groups"] = n.groups;
      d["pad_h"] = n.pad_h;
      d["pad_w"] = n.pad_w;
    }
    if (n.op == wf::OpKind::FoldedConv2d) {
      d["factor"] = n.factor;
      d["bias"] = n.bias;
      d["dtype"] = n.dtype == wf::Dtype::BF16 ? "bf16" : (n.dtype == wf::Dtype::F16 ? "f16" : "tf32");
    }
    d["out_shape"] = n.out_shape;
    out.append(d);
  }
  return out;
}

py::dict cost_dict(const wf::CostEstimate& c) {
  py::dict d;
  d["macs"] = c.macs;
  d["issued_macs"] = c.issued_macs;
  d["aligned"] = c.aligned;
  return d;
}

}  // namespace

PYBIND11_MODULE(_core, m) {
  m.doc() = "widthfold-b200: B200-native width folding for first-layer convolutions";

  py::register_exception<wf::ShapeMismatch>(m, "ShapeMismatchError", PyExc_ValueError);
  py::register_exception<wf::IllegalFold>(m, "IllegalFoldError", PyExc_ValueError);
  py::register_exception<wf::DegenerateOutput>(m, "DegenerateOutputError", PyExc_ValueError);
  py::register_exception<wf::NotBlockDiagonal>(m, "NotBlockDiagonalError", PyExc_RuntimeError);
  py::register_exception<wf::Unsupported>(m, "UnsupportedError", PyExc_RuntimeError);
  py::register_exception<wf::CudaError>(m, "CudaError", PyExc_RuntimeError);

  m.def("abi_version", &wf_abi_version);

  m.def(
      "check_legality",
      [](const wf::Shape& in, const wf::Shape& filt, std::int64_t factor, std::int64_t align, std::int64_t sh,
         std::int64_t sw) { return plan_dict(wf::check_legality(spec_of(in, filt, sh, sw, 0, 0), factor, align)); },
      py::arg("input_shape"), py::arg("filter_shape"), py::arg("factor"), py::arg("align") = 8,
      py::arg("stride_h") = 1, py::arg("stride_w") = 1,
      "Reference fold legality: Apply iff W % F == 0, KW == 1 and stride_w == 1.");

  m.def(
      "choose_fold_factor",
      [](const wf::Shape& in, const wf::Shape& filt, std::int64_t align, std::int64_t sh, std::int64_t sw) {
        return plan_dict(wf::choose_fold_factor(spec_of(in, filt, sh, sw, 0, 0), align));
      },
      py::arg("input_shape"), py::arg("filter_shape"), py::arg("align") = 8, py::arg("stride_h") = 1,
      py::arg("stride_w") = 1, "Smallest factor whose folded channels meet the alignment target.");

  m.def(
      "count_macs",
      [](const wf::Shape& in, const wf::Shape& filt, std::int64_t sh, std::int64_t sw, std::int64_t ph,
         std::int64_t pw) { return wf::count_macs(spec_of(in, filt, sh, sw, ph, pw)).macs; },
      py::arg("input_shape"), py::arg("filter_shape"), py::arg("stride_h") = 1, py::arg("stride_w") = 1,
      py::arg("pad_h") = 0, py::arg("pad_w") = 0);

  m.def(
      "mac_report",
      [](const wf::Shape& in, const wf::Shape& filt, std::int64_t factor, std::int64_t align) {
        const wf::ConvSpec spec = spec_of(in, filt, 1, 1, 0, 0);
        const wf::MacReport r = wf::mac_report(spec, wf::check_legality(spec, factor, align), align);
        py::dict d;
        d["original"] = r.original;
        d["dense_folded"] = r.dense_folded;
        d["grouped_folded"] = r.grouped_folded;
        d["zero_padded"] = r.zero_padded;
        d["factor"] = r.factor;
        return d;
      },
      py::arg("input_shape"), py::arg("filter_shape"), py::arg("factor"), py::arg("align") = 8);

  m.def(
      "plan_fold",
      [](const wf::Shape& in, const wf::Shape& filt, std::int64_t sh, std::int64_t sw, std::int64_t ph,
         std::int64_t pw, std::int64_t factor, std::int64_t group_size, const std::string& dtype) {
        const wf::DevicePlan dp =
            wf::plan_device_fold(spec_of(in, filt, sh, sw, ph, pw), factor, group_size, dtype_of(dtype));
        py::dict d = plan_dict(dp.plan);
        if (dp.plan.ok()) d["device"] = raw_dict(dp.raw);
        return d;
      },
      py::arg("input_shape"), py::arg("filter_shape"), py::arg("stride_h") = 1, py::arg("stride_w") = 1,
      py::arg("pad_h") = 0, py::arg("pad_w") = 0, py::arg("factor") = 0, py::arg("group_size") = 0,
      py::arg("dtype") = "bf16", "Generalized device fold plan (KW > 1, stride, padding).");

  m.def("folded_filter_shape", &wf::folded_filter_shape, py::arg("filter_shape"), py::arg("factor"),
        py::arg("stride_w") = 1, py::arg("pad_w") = 0);

  m.def(
      "conv2d_exact",
      [](std::uintptr_t x, std::uintptr_t w, std::uintptr_t y, const wf::Shape& in, const wf::Shape& filt,
         std::int64_t sh, std::int64_t sw, std::int64_t ph, std::int64_t pw, std::uintptr_t stream) {
        const wf::ConvSpec spec = spec_of(in, filt, sh, sw, ph, pw);
        py::gil_scoped_release nogil;
        wf::conv2d_exact(F(x), F(w), static_cast<float*>(P(y)), spec, P(stream));
      },
      py::arg("x"), py::arg("w"), py::arg("y"), py::arg("input_shape"), py::arg("filter_shape"),
      py::arg("stride_h"), py::arg("stride_w"), py::arg("pad_h"), py::arg("pad_w"), py::arg("stream"));

  m.def(
      "conv2d_grouped",
      [](std::uintptr_t x, std::uintptr_t w, std::uintptr_t y, const wf::Shape& in, const wf::Shape& filt,
         std::int64_t sh, std::int64_t sw, std::int64_t groups, std::uintptr_t stream) {
        const wf::ConvSpec spec = spec_of(in, filt, sh, sw, 0, 0);
        py::gil_scoped_release nogil;
        wf::conv2d_grouped(F(x), F(w), static_cast<float*>(P(y)), spec, groups, P(stream));
      },
      py::arg("x"), py::arg("w"), py::arg("y"), py::arg("input_shape"), py::arg("filter_shape"),
      py::arg("stride_h"), py::arg("stride_w"), py::arg("groups"), py::arg("stream"));

  m.def(
      "bias_add",
      [](std::uintptr_t y, std::uintptr_t b, std::uintptr_t out, std::int64_t n, std::int64_t c, bool relu,
         std::uintptr_t stream) {
        py::gil_scoped_release nogil;
        wf::bias_add(F(y), F(b), static_cast<float*>(P(out)), n, c, relu, P(stream));
      },
      py::arg("y"), py::arg("b"), py::arg("out"), py::arg("n"), py::arg("c"), py::arg("relu"), py::arg("stream"));

  m.def(
      "replicate_bias",
      [](std::uintptr_t b, std::int64_t cout, std::int64_t factor, std::uintptr_t out, std::uintptr_t stream) {
        py::gil_scoped_release nogil;
        wf::replicate_bias(F(b), cout, factor, static_cast<float*>(P(out)), P(stream));
      },
      py::arg("b"), py::arg("cout"), py::arg("factor"), py::arg("out"), py::arg("stream"));

  m.def(
      "expand_filter_general",
      [](std::uintptr_t w, const wf::Shape& fs, std::int64_t factor, std::uintptr_t out, std::uintptr_t stream) {
        py::gil_scoped_release nogil;
        wf::expand_filter_general(F(w), fs, factor, static_cast<float*>(P(out)), P(stream));
      },
      py::arg("w"), py::arg("filter_shape"), py::arg("factor"), py::arg("out"), py::arg("stream"));

  m.def(
      "expand_filter_folded",
      [](std::uintptr_t w, const wf::Shape& fs, std::int64_t factor, std::int64_t sw, std::int64_t pw,
         std::uintptr_t out, std::uintptr_t stream) {
        py::gil_scoped_release nogil;
        wf::expand_filter_folded(F(w), fs, factor, sw, pw, static_cast<float*>(P(out)), P(stream));
      },
      py::arg("w"), py::arg("filter_shape"), py::arg("factor"), py::arg("stride_w"), py::arg("pad_w"),
      py::arg("out"), py::arg("stream"));

  m.def(
      "check_block_diagonal",
      [](std::uintptr_t w, const wf::Shape& s, std::int64_t groups, std::uintptr_t scratch, std::uintptr_t stream) {
        py::gil_scoped_release nogil;
        wf::check_block_diagonal(F(w), s, groups, P(scratch), P(stream));
      },
      py::arg("w"), py::arg("dense_shape"), py::arg("groups"), py::arg("scratch"), py::arg("stream"));

  // ---- model format: tensor bundles + graph JSON (model_io.hpp) ----
  py::register_exception<wf::ManifestParse>(m, "ManifestParseError", PyExc_ValueError);
  py::register_exception<wf::BlobSizeMismatch>(m, "BlobSizeMismatchError", PyExc_ValueError);
  py::register_exception<wf::IoFailure>(m, "IoFailureError", PyExc_OSError);
  m.def(
      "read_bundle",
      [](const std::string& path) {
        const wf::TensorBundle b = wf::read_bundle(path);
        py::list out;
        for (const auto& [name, t] : b.entries())
          out.append(py::make_tuple(name, t.shape, t.dtype,
                                    py::bytes(reinterpret_cast<const char*>(t.bytes.data()), t.bytes.size())));
        return out;
      },
      py::arg("manifest_path"), "[(name, shape, dtype, little-endian bytes)] in manifest order (bundle.hpp:32-36).");
  m.def(
      "write_bundle",
      [](const std::string& path, const py::list& entries) {
        wf::TensorBundle b;
        for (auto h : entries) {
          const py::tuple e = h.cast<py::tuple>();
          wf::BundleTensor t;
          t.shape = e[1].cast<wf::Shape>();
          t.dtype = e[2].cast<std::string>();
          const std::string raw = e[3].cast<std::string>();
          t.bytes.assign(raw.begin(), raw.end());
          b.add(e[0].cast<std::string>(), std::move(t));
        }
        wf::write_bundle(b, path);
      },
      py::arg("manifest_path"), py::arg("entries"), "Write a manifest + <stem>.bin blob (bundle.hpp:38-40).");
  m.def(
      "read_graph",
      [](const std::string& path) {
        const wf::Graph g = wf::read_graph(path);
        py::dict w;
        for (const auto& kv : g.weights) w[py::str(kv.first)] = to_array(kv.second);
        return py::make_tuple(nodes_of(g), w);
      },
      py::arg("path"), "Graph JSON + its weights bundle (graph.hpp:68-70).");
  m.def(
      "write_graph",
      [](const py::list& nodes, const py::dict& weights, const std::string& path) {
        wf::write_graph(graph_of(nodes, weights), path);
      },
      py::arg("nodes"), py::arg("weights"), py::arg("path"));
  py::register_exception<wf::ShapeInferenceFailure>(m, "ShapeInferenceFailureError", PyExc_ValueError);
  py::register_exception<wf::MissingInput>(m, "MissingInputError", PyExc_ValueError);

  m.def(
      "infer_shapes",
      [](const py::list& nodes, const py::dict& weights) { return nodes_of(wf::infer_shapes(graph_of(nodes, weights))); },
      py::arg("nodes"), py::arg("weights"), "Validate a graph and annotate out_shape (graph.hpp).");
  m.def(
      "width_fold_pass",
      [](const py::list& nodes, const py::dict& weights, std::int64_t factor, std::int64_t align,
         const std::string& precision) {
        const wf::FoldFactor ff = factor > 0 ? wf::FoldFactor::fixed(factor) : wf::FoldFactor::automatic();
        wf::PassResult r = wf::width_fold_pass(graph_of(nodes, weights), ff, align, dtype_of(precision));
        py::list decisions;
        for (const auto& d : r.report.decisions) {
          py::dict e;
          e["id"] = d.id;
          e["kind"] = wf::to_string(d.kind);
          e["applied"] = d.applied;
          e["plan"] = plan_dict(d.plan);
          e["note"] = d.note;
          decisions.append(e);
        }
        py::dict report;
        report["decisions"] = decisions;
        report["before"] = cost_dict(r.report.before);
        report["after"] = cost_dict(r.report.after);
        report["applied_count"] = r.report.applied_count();
        py::dict w;
        for (const auto& kv : r.graph.weights) w[py::str(kv.first)] = to_array(kv.second);
        return py::make_tuple(nodes_of(r.graph), w, report);
      },
      py::arg("nodes"), py::arg("weights"), py::arg("factor") = 0, py::arg("align") = 8, py::arg("precision") = "tf32",
      "Rewrite-rule pass (src/pass.cpp:71): every conv2d the device fold applies to becomes folded_conv2d.");
  m.def(
      "interpret",
      [](const py::list& nodes, const py::dict& weights, const py::dict& inputs, const std::string& mode) {
        wf::TensorMap in;
        for (auto item : inputs) in[item.first.cast<std::string>()] = host_tensor(item.second.cast<F32Array>());
        const wf::ExecMode em = mode == "dense" ? wf::ExecMode::Dense
                                : mode == "grouped" ? wf::ExecMode::Grouped
                                                    : wf::ExecMode::Device;
        wf::Graph g = graph_of(nodes, weights);
        wf::TensorMap out;
        {
          py::gil_scoped_release nogil;
          out = wf::interpret(g, in, em);
        }
        py::dict d;
        for (const auto& kv : out) d[py::str(kv.first)] = to_array(kv.second);
        return d;
      },
      py::arg("nodes"), py::arg("weights"), py::arg("inputs"), py::arg("mode") = "device",
      "Execute the graph on the GPU (src/interpreter.cpp:8).");

  py::class_<wf::FoldedConv>(m, "FoldedConv")
      .def(py::init([](const wf::Shape& in, const wf::Shape& filt, std::int64_t sh, std::int64_t sw,
                       std::int64_t ph, std::int64_t pw, const std::string& dtype, std::int64_t factor,
                       std::int64_t group_size, const std::string& variant) {
             if (variant != "fold" && variant != "unfolded")
               throw std::invalid_argument("variant must be 'fold' or 'unfolded'");
             return wf::FoldedConv(spec_of(in, filt, sh, sw, ph, pw), dtype_of(dtype), factor, group_size,
                                   variant == "unfolded" ? wf::FoldedConv::Variant::Unfolded
                                                         : wf::FoldedConv::Variant::Fold);
           }),
           py::arg("input_shape"), py::arg("filter_shape"), py::arg("stride_h") = 1, py::arg("stride_w") = 1,
           py::arg("pad_h") = 0, py::arg("pad_w") = 0, py::arg("dtype") = "bf16", py::arg("factor") = 0,
           py::arg("group_size") = 0, py::arg("variant") = "fold")
      .def_property_readonly("packed_bytes", &wf::FoldedConv::packed_bytes)
      .def_property_readonly("cout_f", &wf::FoldedConv::cout_f)
      .def_property_readonly("plan", [](const wf::FoldedConv& c) { return plan_dict(c.plan()); })
      .def_property_readonly("device", [](const wf::FoldedConv& c) { return raw_dict(c.raw()); })
      .def_property_readonly("output_shape", [](const wf::FoldedConv& c) { return c.spec().output_shape(); })
      .def(
          "pack",
          [](const wf::FoldedConv& c, std::uintptr_t w, std::uintptr_t b, std::uintptr_t packed, std::uintptr_t brep,
             std::uintptr_t stream) {
            py::gil_scoped_release nogil;
            c.pack(P(w), b ? F(b) : nullptr, P(packed), brep ? static_cast<float*>(P(brep)) : nullptr, P(stream));
          },
          py::arg("w"), py::arg("b"), py::arg("packed"), py::arg("b_rep"), py::arg("stream"))
      .def(
          "forward",
          [](const wf::FoldedConv& c, std::uintptr_t x, std::uintptr_t packed, std::uintptr_t brep, std::uintptr_t y,
             const std::string& out_dtype, bool bias, bool relu, std::uintptr_t stream, std::uint32_t flags,
             std::uintptr_t workspace) {
            const wf::Dtype od = dtype_of(out_dtype);
            py::gil_scoped_release nogil;
            c.forward(P(x), P(packed), brep ? F(brep) : nullptr, P(y), od, bias, relu, P(stream), flags,
                      workspace ? P(workspace) : nullptr);
          },
          py::arg("x"), py::arg("packed"), py::arg("b_rep"), py::arg("y"), py::arg("out_dtype"), py::arg("bias"),
          py::arg("relu"), py::arg("stream"), py::arg("extra_flags") = 0, py::arg("workspace") = 0)
      .def(
          "repitch",
          [](const wf::FoldedConv& c, std::uintptr_t x, std::uintptr_t workspace, std::uintptr_t stream) {
            py::gil_scoped_release nogil;
            c.repitch(P(x), workspace ? P(workspace) : nullptr, P(stream));
          },
          py::arg("x"), py::arg("workspace"), py::arg("stream"))
      .def_property_readonly("workspace_bytes", &wf::FoldedConv::workspace_bytes);
}
