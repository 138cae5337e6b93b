// mgrx_b200.hpp — C++ drop-in for the reference's hot-path entry points.
//
// Include this next to the reference's own headers (proj/core/include) and
// link libmgrx_b200.so.  Every function keeps the reference's signature and
// error behaviour but runs on the B200 through the C-ABI (mgrx_b200.h):
//
//   reference                                      drop-in
//   mgrx::decompose        (transform.hpp:509)     mgrx::b200::decompose
//   mgrx::decompose_with   (transform.hpp:486)     mgrx::b200::decompose_with (level by level; the decider runs on the host)
//   mgrx::recompose        (transform.hpp:517)     mgrx::b200::recompose
//   mgrx::quantize         (quantize.hpp:79)       mgrx::b200::quantize
//   mgrx::quantize_tail    (quantize.hpp:99)       mgrx::b200::quantize_tail
//   mgrx::dequantize       (quantize.hpp:118)      mgrx::b200::dequantize
//   mgrx::dequantize_tail  (quantize.hpp:137)      mgrx::b200::dequantize_tail
//   mgrx::compress         (pipeline.hpp:130)      mgrx::b200::compress   (fixed, forced or adaptive stop; the
//                                                   adaptive decider runs on the GPU: decompose_adaptive)
//   mgrx::decompress_field (pipeline.hpp:198)      mgrx::b200::decompress_field
//   mgrx::SolverWorkspace  (transform.hpp:48)      mgrx::b200::Workspace  (owns the GPU context)
//
// Status codes from the C-ABI are rethrown as mgrx::Error with the same
// errc (error.hpp:9-36); CUDA failures become errc::invalid_input with the
// CUDA message.  The lossless back end (Huffman, container) stays the
// reference's own host code.
#ifndef MGRX_B200_HPP
#define MGRX_B200_HPP

#include <algorithm>
#include <cstdint>
#include <optional>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "mgrx/pipeline.hpp"
#include "mgrx/quantize.hpp"
#include "mgrx/transform.hpp"
#include "mgrx_b200.h"

namespace mgrx::b200 {

inline void check(int status, const mgrx_gpu_ctx* ctx = nullptr) {
  if (status == MGRX_OK) return;
  const std::string msg = ctx ? mgrx_gpu_last_error(ctx) : "mgrx_b200 error";
  if (status >= 1 && status <= 15) fail(static_cast<errc>(status - 1), msg);
  fail(errc::invalid_input, "mgrx_b200 status " + std::to_string(status) + ": " + msg);
}

// GPU analogue of SolverWorkspace: one per host thread.
class Workspace {
 public:
  explicit Workspace(int device = 0) { check(mgrx_gpu_ctx_create(device, &ctx_)); }
  Workspace(const Workspace&) = delete;
  Workspace& operator=(const Workspace&) = delete;
  ~Workspace() { mgrx_gpu_ctx_destroy(ctx_); }
  mgrx_gpu_ctx* get() const { return ctx_; }
  void prepare(const GridHierarchy&) {}

 private:
  mgrx_gpu_ctx* ctx_ = nullptr;
};

namespace detail {
template <typename T>
constexpr int dtype() {
  return sizeof(T) == 4 ? MGRX_F32 : MGRX_F64;
}
inline std::vector<uint64_t> dims64(const Dims& d) { return std::vector<uint64_t>(d.begin(), d.end()); }
}  // namespace detail

template <typename T>
MultilevelCoefficients<T> decompose(TensorField<T> field, const GridHierarchy& h, int stop_level, Workspace& ws) {
  if (field.dims != h.level_dims(h.num_levels())) fail(errc::shape_error, "field dims do not match hierarchy");
  if (stop_level < 0 || stop_level > h.num_levels()) fail(errc::invalid_level, "stop level out of range");
  const auto d = detail::dims64(field.dims);
  MultilevelCoefficients<T> out{std::vector<T>(field.size()), h, stop_level};
  check(mgrx_host_decompose(ws.get(), detail::dtype<T>(), int(d.size()), d.data(), h.num_levels(), stop_level,
                            field.data.data(), out.buffer.data()),
        ws.get());
  return out;
}

// decompose_with (transform.hpp:485-506): before each level the decider sees
// that level's block (natural order) and may stop the recursion there.  The
// level steps run on the GPU one at a time (the level block decomposed as a
// field of `l` levels, stopped at l - 1 — the same arithmetic as the full
// decompose); each step's coarse block comes back to the host for the next
// decision.
template <typename T>
MultilevelCoefficients<T> decompose_with(TensorField<T> field, const GridHierarchy& h, Workspace& ws,
                                         const StopDecider<T>& decider, int min_stop_level = 0) {
  const int L = h.num_levels();
  if (field.dims != h.level_dims(L)) fail(errc::shape_error, "field dims do not match hierarchy");
  if (min_stop_level < 0 || min_stop_level > L) fail(errc::invalid_level, "stop level out of range");
  if (!decider) return decompose(std::move(field), h, min_stop_level, ws);
  std::vector<T> out(h.total_count());
  std::vector<T> block = std::move(field.data);  // level-l block, natural order
  int stop = min_stop_level;
  for (int l = L; l > min_stop_level; --l) {
    const Dims dl = h.level_dims(l);
    if (decider(l, BlockView<const T>{block.data(), dl, row_major_strides(dl)})) {
      stop = l;
      break;
    }
    const auto d = detail::dims64(dl);
    std::vector<T> step(h.node_count(l));  // [coarse block of l - 1 | shell of level l]
    check(mgrx_host_decompose(ws.get(), detail::dtype<T>(), int(d.size()), d.data(), l, l - 1, block.data(),
                              step.data()),
          ws.get());
    const std::ptrdiff_t nc = static_cast<std::ptrdiff_t>(h.node_count(l - 1));
    std::copy(step.begin() + nc, step.end(), out.begin() + nc);
    block.assign(step.begin(), step.begin() + nc);
  }
  std::copy(block.begin(), block.end(), out.begin());  // coarse block of the stop level
  return MultilevelCoefficients<T>{std::move(out), h, stop};
}

template <typename T>
TensorField<T> recompose(const MultilevelCoefficients<T>& coeffs, Workspace& ws) {
  const GridHierarchy& h = coeffs.hierarchy;
  if (coeffs.buffer.size() != h.total_count()) fail(errc::shape_error, "buffer size != total node count");
  TensorField<T> f(h.level_dims(h.num_levels()));
  const auto d = detail::dims64(f.dims);
  check(mgrx_host_recompose(ws.get(), detail::dtype<T>(), int(d.size()), d.data(), h.num_levels(), coeffs.stop_level,
                            coeffs.buffer.data(), f.data.data()),
        ws.get());
  return f;
}

namespace detail {
template <typename T>
LabelStream<T> quantize_impl(std::span<const T> buffer, const GridHierarchy& h, int stop, const QuantizationPlan& plan,
                             Workspace& ws) {
  if (plan.num_levels() != h.num_levels()) fail(errc::shape_error, "plan does not match hierarchy");
  const auto d = dims64(h.level_dims(h.num_levels()));
  const size_t base = stop == 0 ? 0 : h.node_count(stop);
  std::vector<int32_t> flat(h.total_count() - base);
  uint64_t cap = 1 << 16, n = 0;
  std::vector<uint64_t> pos;
  std::vector<T> val;
  for (;;) {
    pos.resize(cap);
    val.resize(cap);
    const int rc = mgrx_host_quantize(ws.get(), dtype<T>(), int(d.size()), d.data(), h.num_levels(), stop,
                                      plan.bin_widths.data(), buffer.data(), flat.data(), pos.data(), val.data(), cap,
                                      &n);
    if (rc == MGRX_CAPACITY_EXCEEDED) {
      cap = n;
      continue;
    }
    check(rc, ws.get());
    break;
  }
  LabelStream<T> s;
  size_t at = 0;
  for (int l = stop == 0 ? 0 : stop + 1; l <= h.num_levels(); ++l) {
    s.labels.emplace_back(flat.begin() + std::ptrdiff_t(at), flat.begin() + std::ptrdiff_t(at + h.delta_count(l)));
    at += h.delta_count(l);
  }
  s.outliers.reserve(n);
  for (uint64_t i = 0; i < n; ++i) s.outliers.push_back({pos[i], val[i]});
  return s;
}

template <typename T>
void dequantize_impl(std::span<T> buffer, const LabelStream<T>& stream, const GridHierarchy& h, int stop,
                     const QuantizationPlan& plan, Workspace& ws) {
  const int first = stop == 0 ? 0 : stop + 1;
  if (stream.labels.size() != size_t(h.num_levels() + 1 - first))
    fail(errc::shape_error, "label stream does not match hierarchy");
  std::vector<int32_t> flat;
  for (int l = first; l <= h.num_levels(); ++l) {
    const auto& lv = stream.labels[size_t(l - first)];
    if (lv.size() != h.delta_count(l)) fail(errc::shape_error, "label count mismatch");
    flat.insert(flat.end(), lv.begin(), lv.end());
  }
  std::vector<uint64_t> pos;
  std::vector<T> val;
  for (const auto& o : stream.outliers) {
    pos.push_back(o.position);
    val.push_back(o.value);
  }
  const auto d = dims64(h.level_dims(h.num_levels()));
  check(mgrx_host_dequantize(ws.get(), dtype<T>(), int(d.size()), d.data(), h.num_levels(), stop,
                             plan.bin_widths.data(), flat.data(), pos.data(), val.data(), pos.size(), buffer.data()),
        ws.get());
}
// dequantize (+ the decoded coarse block for a tail stream) + recompose in
// one device-resident pass (mgrx_host_decompress): the coefficients never
// come back to the host.
template <typename T>
TensorField<T> decompress_impl(const LabelStream<T>& stream, const GridHierarchy& h, int stop,
                               const QuantizationPlan& plan, const T* coarse, Workspace& ws) {
  const int first = stop == 0 ? 0 : stop + 1;
  if (stream.labels.size() != size_t(h.num_levels() + 1 - first))
    fail(errc::shape_error, "label stream does not match hierarchy");
  std::vector<int32_t> flat;
  flat.reserve(h.total_count());
  for (int l = first; l <= h.num_levels(); ++l) {
    const auto& lv = stream.labels[size_t(l - first)];
    if (lv.size() != h.delta_count(l)) fail(errc::shape_error, "label count mismatch");
    flat.insert(flat.end(), lv.begin(), lv.end());
  }
  std::vector<uint64_t> pos;
  std::vector<T> val;
  for (const auto& o : stream.outliers) {
    pos.push_back(o.position);
    val.push_back(o.value);
  }
  TensorField<T> out;
  out.dims = h.level_dims(h.num_levels());
  out.data.resize(h.total_count());
  const auto d = dims64(out.dims);
  check(mgrx_host_decompress(ws.get(), dtype<T>(), int(d.size()), d.data(), h.num_levels(), stop,
                             plan.bin_widths.data(), flat.data(), pos.data(), val.data(), pos.size(), coarse,
                             out.data.data()),
        ws.get());
  return out;
}
}  // namespace detail

template <typename T>
LabelStream<T> quantize(const MultilevelCoefficients<T>& coeffs, const QuantizationPlan& plan, Workspace& ws) {
  if (coeffs.stop_level != 0) fail(errc::invalid_input, "quantize expects a fully decomposed buffer");
  return detail::quantize_impl<T>(coeffs.buffer, coeffs.hierarchy, 0, plan, ws);
}

template <typename T>
LabelStream<T> quantize_tail(std::span<const T> buffer, const GridHierarchy& h, int stop_level,
                             const QuantizationPlan& plan, Workspace& ws) {
  return detail::quantize_impl<T>(buffer, h, stop_level, plan, ws);
}

template <typename T>
MultilevelCoefficients<T> dequantize(const LabelStream<T>& stream, const QuantizationPlan& plan, const GridHierarchy& h,
                                     Workspace& ws) {
  MultilevelCoefficients<T> out{std::vector<T>(h.total_count()), h, 0};
  detail::dequantize_impl<T>(out.buffer, stream, h, 0, plan, ws);
  return out;
}

template <typename T>
void dequantize_tail(std::span<T> buffer, const LabelStream<T>& stream, const GridHierarchy& h, int stop_level,
                     const QuantizationPlan& plan, Workspace& ws) {
  detail::dequantize_impl<T>(buffer, stream, h, stop_level, plan, ws);
}

// decompose_with + the reference's adaptive decider (compress,
// pipeline.hpp:148-156) with the level blocks kept on the GPU: the
// per-level penalty models come from the reference's penalty_model_for
// (adaptive.cpp:55-72, host, cached); choose_stop's sampled estimate runs on
// the GPU (mgrx_host_decompose_adaptive, bit-identical totals).
template <typename T>
MultilevelCoefficients<T> decompose_adaptive(const TensorField<T>& field, const GridHierarchy& h,
                                             const QuantizationPlan& plan, std::uint64_t seed, Workspace& ws) {
  const int L = h.num_levels();
  const int d = static_cast<int>(field.dims.size());
  std::vector<double> e(L + 1, 0.0), pen(size_t(L + 1) * d, 0.0), lz(L + 1, 0.0);
  for (int l = 1; l <= L; ++l) {
    e[l] = plan.bin_widths[static_cast<std::size_t>(l)] / 2.0;
    const double kappa = plan.bin_widths[static_cast<std::size_t>(l)] / plan.bin_widths[static_cast<std::size_t>(l - 1)];
    const PenaltyModel& m = penalty_model_for(d, kappa, seed);
    if (static_cast<int>(m.interp.size()) < d) fail(errc::invalid_input, "penalty model rank too small");
    for (int i = 0; i < d; ++i) pen[size_t(l) * d + i] = m.interp[static_cast<std::size_t>(i)];
    lz[l] = m.lorenzo;
  }
  const auto dd = detail::dims64(field.dims);
  std::vector<T> out(h.total_count());
  int stop = 0;
  check(mgrx_host_decompose_adaptive(ws.get(), detail::dtype<T>(), d, dd.data(), L, field.data.data(), e.data(),
                                     pen.data(), lz.data(), 8, 0, out.data(), &stop),
        ws.get());
  return MultilevelCoefficients<T>{std::move(out), h, stop};
}

// compress (pipeline.hpp:130-196) device-resident: the field is copied to
// the GPU once; the adaptive stop decision (choose_stop, adaptive.hpp:99-104),
// decompose, quantize and the labels' entropy coding (encode_labels,
// huffman.cpp:209-255) run there (mgrx_host_compress), and the Lorenzo coder
// of the coarse block too (lorenzo_section_gpu); the reference's container
// assembles the artifact on the host.
// lorenzo_section (pipeline.hpp:86-96) of compress_lorenzo(block, e)
// (lorenzo.hpp:87-128) with the coder and its label entropy coding on the
// GPU (mgrx_host_lorenzo, bit-identical); large blocks (> 2^24 values, the
// one-CTA wavefront's limit of usefulness) use the reference's host coder.
template <typename T>
std::vector<std::uint8_t> lorenzo_section_gpu(const TensorField<T>& block, double e, Workspace& ws) {
  const std::size_t N = block.size();
  if (N > (std::size_t(1) << 24)) return mgrx::detail::lorenzo_section(compress_lorenzo(block, e));
  const auto dd = detail::dims64(block.dims);
  std::vector<std::uint8_t> enc(16 + (1u << 17) + 4 * N + 64);
  std::uint64_t enc_size = 0, cap = std::max<std::uint64_t>(1u << 12, N / 64), nout = 0;
  std::vector<std::uint64_t> pos;
  std::vector<T> val;
  for (;;) {
    pos.resize(cap);
    val.resize(cap);
    const int rc = mgrx_host_lorenzo(ws.get(), detail::dtype<T>(), int(dd.size()), dd.data(), block.data.data(), e,
                                     enc.data(), enc.size(), &enc_size, pos.data(), val.data(), cap, &nout);
    if (rc == MGRX_CAPACITY_EXCEEDED && nout > cap) {
      cap = nout;
      continue;
    }
    check(rc, ws.get());
    break;
  }
  ByteWriter w;
  w.f64(e);
  w.u64(N);
  w.u64(enc_size);
  w.raw(std::span<const std::uint8_t>(enc.data(), enc_size));
  std::vector<Outlier<T>> outliers;
  outliers.reserve(nout);
  for (std::uint64_t i = 0; i < nout; ++i) outliers.push_back({pos[i], val[i]});
  mgrx::detail::write_outliers(w, outliers);
  return std::move(w.bytes);
}

template <typename T>
std::vector<std::uint8_t> compress(const TensorField<T>& field, const CompressOptions& opt, Workspace& ws) {
  // check_finite (pipeline.hpp:132) runs on the GPU inside mgrx_host_compress
  const GridHierarchy h = GridHierarchy::create(field.dims, opt.levels);
  const int L = h.num_levels();
  const QuantizationPlan plan = make_plan(opt.quant_mode, opt.budget, h);
  if (opt.force_stop_level && (*opt.force_stop_level < 0 || *opt.force_stop_level > L))
    fail(errc::invalid_level, "forced stop level out of range");
  const bool adaptive = !opt.force_stop_level && opt.adaptive;
  const int d = static_cast<int>(field.dims.size());
  // per-level penalty tables of the adaptive decision (penalty_model_for, host)
  std::vector<double> e(L + 1, 0.0), pen(size_t(L + 1) * d, 0.0), lz(L + 1, 0.0);
  if (adaptive)
    for (int l = 1; l <= L; ++l) {
      e[l] = plan.bin_widths[static_cast<std::size_t>(l)] / 2.0;
      const double kappa =
          plan.bin_widths[static_cast<std::size_t>(l)] / plan.bin_widths[static_cast<std::size_t>(l - 1)];
      const PenaltyModel& m = penalty_model_for(d, kappa, opt.seed);
      if (static_cast<int>(m.interp.size()) < d) fail(errc::invalid_input, "penalty model rank too small");
      for (int i = 0; i < d; ++i) pen[size_t(l) * d + i] = m.interp[static_cast<std::size_t>(i)];
      lz[l] = m.lorenzo;
    }
  // decompose + quantize + encode_labels on the GPU (mgrx_host_compress);
  // only the encoded sections, the outliers and the coarse block return
  const auto dd = detail::dims64(field.dims);
  const size_t N = h.total_count();
  std::vector<std::uint8_t> sec(4 * N + size_t(L + 1) * (16 + (1u << 17)) + 64);
  std::vector<std::uint64_t> sec_sizes(L + 1, 0);
  std::vector<std::uint64_t> opos;
  std::vector<T> oval, coarse(N);
  std::uint64_t cap = std::max<std::uint64_t>(1u << 16, N / 64), nout = 0;
  int stop = 0;
  for (;;) {
    opos.resize(cap);
    oval.resize(cap);
    const int rc = mgrx_host_compress(ws.get(), detail::dtype<T>(), d, dd.data(), L, field.data.data(),
                                      plan.bin_widths.data(), adaptive ? 1 : 0,
                                      opt.force_stop_level ? *opt.force_stop_level : -1, e.data(), pen.data(),
                                      lz.data(), sec.data(), sec.size(), sec_sizes.data(), opos.data(), oval.data(),
                                      cap, &nout, coarse.data(), &stop);
    if (rc == MGRX_CAPACITY_EXCEEDED && nout > cap) {
      cap = nout;
      continue;
    }
    check(rc, ws.get());
    break;
  }
  Artifact a;
  a.element_type = element_type_of<T>();
  a.dims = field.dims;
  a.levels = static_cast<std::uint8_t>(L);
  a.stop_level = static_cast<std::uint8_t>(stop);
  a.quant_mode = plan.mode;
  a.budget = plan.budget;
  a.bin_widths = plan.bin_widths;
  if (stop == L) {
    a.method = Method::lorenzo_only;
    a.sections.push_back(lorenzo_section_gpu(field, opt.budget, ws));
    return write_artifact(a);
  }
  // label sections: u64 count + encode_labels bytes (label_section, pipeline.hpp:69-75)
  std::size_t at = 0;
  for (int l = stop == 0 ? 0 : stop + 1; l <= L; ++l) {
    ByteWriter w;
    w.u64(h.delta_count(l));
    w.raw(std::span<const std::uint8_t>(sec.data() + at, sec_sizes[static_cast<std::size_t>(l)]));
    at += sec_sizes[static_cast<std::size_t>(l)];
    a.sections.push_back(std::move(w.bytes));
  }
  std::vector<Outlier<T>> outliers;
  outliers.reserve(nout);
  for (std::uint64_t i = 0; i < nout; ++i) outliers.push_back({opos[i], oval[i]});
  ByteWriter w;
  mgrx::detail::write_outliers(w, outliers);
  a.sections.push_back(std::move(w.bytes));
  if (stop == 0) {
    a.method = Method::multigrid_full;
  } else {
    a.method = Method::multigrid_lorenzo;
    coarse.resize(h.node_count(stop));
    TensorField<T> cf(h.level_dims(stop), std::move(coarse));
    a.sections.push_back(lorenzo_section_gpu(cf, coarse_error_bound(plan, stop), ws));
  }
  return write_artifact(a);
}

// decompress_field (pipeline.hpp:198-261) with dequantize + recompose on
// the GPU.
template <typename T>
TensorField<T> decompress_field(const Artifact& a, Workspace& ws) {
  if (a.element_type != element_type_of<T>()) fail(errc::invalid_input, "element type mismatch");
  const GridHierarchy h = GridHierarchy::create(a.dims, static_cast<int>(a.levels));
  const int L = h.num_levels();
  const int stop = a.stop_level;
  if (a.method == Method::lorenzo_only) return mgrx::decompress_field<T>(a);
  for (double q : a.bin_widths)
    if (!(q > 0.0) || !std::isfinite(q)) fail(errc::corrupt, "bad bin width");
  QuantizationPlan plan;
  plan.mode = a.quant_mode;
  plan.budget = a.budget;
  plan.bin_widths = a.bin_widths;
  if (a.method == Method::multigrid_full) {
    if (stop != 0) fail(errc::corrupt, "bad stop level for full method");
    if (a.sections.size() != static_cast<std::size_t>(L) + 2) fail(errc::corrupt, "unexpected section count");
    LabelStream<T> stream;
    stream.labels.resize(static_cast<std::size_t>(L) + 1);
    for (int l = 0; l <= L; ++l)
      stream.labels[static_cast<std::size_t>(l)] =
          mgrx::detail::parse_label_section(a.sections[static_cast<std::size_t>(l)], h.delta_count(l));
    ByteReader r{a.sections.back()};
    stream.outliers = mgrx::detail::read_outliers<T>(r, h.total_count());
    return detail::decompress_impl<T>(stream, h, 0, plan, nullptr, ws);
  }
  if (stop < 1 || stop > L) fail(errc::corrupt, "bad stop level");
  const std::size_t tail_levels = static_cast<std::size_t>(L - stop);
  if (a.sections.size() != tail_levels + 2) fail(errc::corrupt, "unexpected section count");
  LabelStream<T> stream;
  stream.labels.resize(tail_levels);
  for (std::size_t i = 0; i < tail_levels; ++i)
    stream.labels[i] =
        mgrx::detail::parse_label_section(a.sections[i], h.delta_count(stop + 1 + static_cast<int>(i)));
  {
    ByteReader r{a.sections[tail_levels]};
    stream.outliers = mgrx::detail::read_outliers<T>(r, h.total_count());
    for (const auto& o : stream.outliers)
      if (o.position < h.node_count(stop)) fail(errc::corrupt, "outlier inside coarse block");
  }
  LorenzoStream<T> coarse_stream = mgrx::detail::parse_lorenzo_section<T>(a.sections.back(), h.node_count(stop));
  TensorField<T> coarse = decompress_lorenzo(coarse_stream, h.level_dims(stop));
  return detail::decompress_impl<T>(stream, h, stop, plan, coarse.data.data(), ws);
}

}  // namespace mgrx::b200

#endif  // MGRX_B200_HPP
