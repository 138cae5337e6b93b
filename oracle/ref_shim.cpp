// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference implementation
// (/root/reference/proj/core, compiled from its own sources by
// oracle/Makefile into oracle/_ref/libmgrx_ref.so).  It lets the Python
// tests, the golden-fixture generator and bench.py's CPU-baseline arm call
// the reference's own decompose / recompose / quantize / dequantize
// (transform.hpp:509,517; quantize.hpp:79,118) and its component kernels on
// plain buffers.  Every function returns 0 on success or 1 + mgrx::errc on a
// reference exception (error.hpp:9-36), 99 on anything else.
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <span>
#include <vector>

#include "mgrx/adaptive.hpp"
#include "mgrx/grid.hpp"
#include "mgrx/huffman.hpp"
#include "mgrx/lorenzo.hpp"
#include "mgrx/quantize.hpp"
#include "mgrx/reference.hpp"
#include "mgrx/reorder.hpp"
#include "mgrx/transform.hpp"

namespace {

thread_local char g_msg[512];

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_msg[0] = 0;
    return 0;
  } catch (const mgrx::Error& e) {
    std::strncpy(g_msg, e.what(), sizeof(g_msg) - 1);
    return 1 + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    std::strncpy(g_msg, e.what(), sizeof(g_msg) - 1);
    return 99;
  }
}

mgrx::Dims to_dims(int nd, const uint64_t* dims) {
  mgrx::Dims d(static_cast<std::size_t>(nd));
  for (int i = 0; i < nd; ++i) d[static_cast<std::size_t>(i)] = dims[i];
  return d;
}

mgrx::GridHierarchy hier(int nd, const uint64_t* dims, int levels) {
  return levels < 0 ? mgrx::GridHierarchy::create(to_dims(nd, dims))
                    : mgrx::GridHierarchy::create(to_dims(nd, dims), levels);
}

template <typename T>
int decompose_t(int nd, const uint64_t* dims, int levels, int stop, const T* in, T* out,
                int batch) {
  return guarded([&] {
    mgrx::GridHierarchy h = hier(nd, dims, levels);
    mgrx::TensorField<T> f(to_dims(nd, dims));
    std::memcpy(f.data.data(), in, f.size() * sizeof(T));
    mgrx::SolverWorkspace ws(static_cast<std::size_t>(batch));
    ws.prepare(h);
    mgrx::MultilevelCoefficients<T> mc = mgrx::decompose(std::move(f), h, stop, ws);
    std::memcpy(out, mc.buffer.data(), mc.buffer.size() * sizeof(T));
  });
}

template <typename T>
int recompose_t(int nd, const uint64_t* dims, int levels, int stop, const T* in, T* out) {
  return guarded([&] {
    mgrx::GridHierarchy h = hier(nd, dims, levels);
    mgrx::MultilevelCoefficients<T> mc{std::vector<T>(in, in + h.total_count()), h, stop};
    mgrx::SolverWorkspace ws;
    ws.prepare(h);
    mgrx::TensorField<T> f = mgrx::recompose(mc, ws);
    std::memcpy(out, f.data.data(), f.size() * sizeof(T));
  });
}

template <typename T>
int strided_decompose_t(int nd, const uint64_t* dims, int levels, int stop, const T* in, T* out) {
  return guarded([&] {
    mgrx::GridHierarchy h = hier(nd, dims, levels);
    mgrx::TensorField<T> f(to_dims(nd, dims));
    std::memcpy(f.data.data(), in, f.size() * sizeof(T));
    mgrx::MultilevelCoefficients<T> mc = mgrx::reference_decompose(std::move(f), h, stop);
    std::memcpy(out, mc.buffer.data(), mc.buffer.size() * sizeof(T));
  });
}

// quantize (stop == 0) or quantize_tail (stop > 0).  labels: concatenated
// per-level label vectors; outliers written up to `cap`, *n_out = count.
template <typename T>
int quantize_t(int nd, const uint64_t* dims, int levels, int stop, const double* q, const T* coeffs,
               int32_t* labels, uint64_t* opos, T* oval, uint64_t cap, uint64_t* n_out) {
  return guarded([&] {
    mgrx::GridHierarchy h = hier(nd, dims, levels);
    mgrx::QuantizationPlan plan;
    plan.bin_widths.assign(q, q + h.num_levels() + 1);
    mgrx::LabelStream<T> s;
    if (stop == 0) {
      mgrx::MultilevelCoefficients<T> mc{std::vector<T>(coeffs, coeffs + h.total_count()), h, 0};
      s = mgrx::quantize(mc, plan);
    } else {
      s = mgrx::quantize_tail<T>(std::span<const T>(coeffs, h.total_count()), h, stop, plan);
    }
    std::size_t pos = 0;
    for (const auto& lv : s.labels) {
      std::memcpy(labels + pos, lv.data(), lv.size() * sizeof(int32_t));
      pos += lv.size();
    }
    *n_out = s.outliers.size();
    for (std::size_t i = 0; i < s.outliers.size() && i < cap; ++i) {
      opos[i] = s.outliers[i].position;
      oval[i] = s.outliers[i].value;
    }
  });
}

template <typename T>
int dequantize_t(int nd, const uint64_t* dims, int levels, int stop, const double* q,
                 const int32_t* labels, const uint64_t* opos, const T* oval, uint64_t n_out,
                 T* coeffs) {
  return guarded([&] {
    mgrx::GridHierarchy h = hier(nd, dims, levels);
    mgrx::QuantizationPlan plan;
    plan.bin_widths.assign(q, q + h.num_levels() + 1);
    mgrx::LabelStream<T> s;
    std::size_t lp = 0;  // labels are the concatenated per-level vectors
    for (int l = stop == 0 ? 0 : stop + 1; l <= h.num_levels(); ++l) {
      s.labels.emplace_back(labels + lp, labels + lp + h.delta_count(l));
      lp += h.delta_count(l);
    }
    for (uint64_t i = 0; i < n_out; ++i) s.outliers.push_back({opos[i], oval[i]});
    if (stop == 0) {
      mgrx::MultilevelCoefficients<T> mc = mgrx::dequantize(s, plan, h);
      std::memcpy(coeffs, mc.buffer.data(), mc.buffer.size() * sizeof(T));
    } else {
      mgrx::dequantize_tail<T>(std::span<T>(coeffs, h.total_count()), s, h, stop, plan);
    }
  });
}

// One level step of decompose at `level` on a field already holding the
// level block in natural order (corner of the full array): returns the
// reordered+coefficient field (the state after compute_coefficients) and the
// correction (coarse extents, row-major packed).
template <typename T>
int level_step_t(int nd, const uint64_t* dims, int level, T* field, double* corr_out) {
  return guarded([&] {
    mgrx::GridHierarchy h = hier(nd, dims, -1);
    mgrx::TensorField<T> f(to_dims(nd, dims));
    std::memcpy(f.data.data(), field, f.size() * sizeof(T));
    mgrx::reorder_level(f, h, level);
    mgrx::compute_coefficients(f, h, level);
    mgrx::SolverWorkspace ws;
    mgrx::Correction c = mgrx::compute_correction(f, h, level, ws);
    std::memcpy(field, f.data.data(), f.size() * sizeof(T));
    // pack the correction (strides are those of the level extents)
    const int d = nd;
    std::vector<std::size_t> idx(static_cast<std::size_t>(d), 0);
    const std::size_t total = mgrx::element_count(c.extents);
    for (std::size_t p = 0; p < total; ++p) {
      std::size_t off = 0;
      for (int i = 0; i < d; ++i) off += idx[static_cast<std::size_t>(i)] * c.strides[static_cast<std::size_t>(i)];
      corr_out[p] = c.data[off];
      for (int i = d - 1; i >= 0; --i) {
        if (++idx[static_cast<std::size_t>(i)] < c.extents[static_cast<std::size_t>(i)]) break;
        idx[static_cast<std::size_t>(i)] = 0;
      }
    }
  });
}

// The adaptive stop decision's sampled totals (accumulate_block_errors,
// adaptive.hpp:51-94) and decision (choose_stop, :99-104).
template <typename T>
int choose_stop_t(int nd, const uint64_t* dims, const T* data, double e, const double* interp_pen,
                  double lorenzo_pen, int step, double* totals, int* stop) {
  return guarded([&] {
    const mgrx::Dims dl = to_dims(nd, dims);
    mgrx::BlockView<const T> v{data, dl, mgrx::row_major_strides(dl)};
    mgrx::PenaltyModel m;
    m.lorenzo = lorenzo_pen;
    m.interp.assign(interp_pen, interp_pen + nd);
    mgrx::BlockErrors total;
    const bool any = mgrx::detail::accumulate_block_errors(v, static_cast<std::size_t>(step), e, m, total);
    totals[0] = total.lorenzo;
    totals[1] = total.interp;
    *stop = any ? (total.lorenzo < total.interp ? 1 : 0) : 1;
  });
}

// compress_lorenzo (lorenzo.hpp:87-128): labels, outliers.
template <typename T>
int lorenzo_t(int nd, const uint64_t* dims, const T* data, double e, int32_t* labels, uint64_t* opos, T* oval,
              uint64_t cap, uint64_t* n_out) {
  return guarded([&] {
    mgrx::TensorField<T> f(to_dims(nd, dims));
    std::memcpy(f.data.data(), data, f.size() * sizeof(T));
    const mgrx::LorenzoStream<T> s = mgrx::compress_lorenzo(f, e);
    std::memcpy(labels, s.labels.data(), s.labels.size() * 4);
    *n_out = s.outliers.size();
    if (s.outliers.size() > cap) mgrx::fail(mgrx::errc::invalid_input, "capacity");
    for (std::size_t i = 0; i < s.outliers.size(); ++i) {
      opos[i] = s.outliers[i].position;
      oval[i] = s.outliers[i].value;
    }
  });
}

} // namespace

extern "C" {

// encode_labels (huffman.hpp:14, src/huffman.cpp:209-255).
int ref_encode_labels(const int32_t* labels, uint64_t n, uint8_t* out, uint64_t cap, uint64_t* size) {
  return guarded([&] {
    const std::vector<std::uint8_t> b = mgrx::encode_labels(std::span<const std::int32_t>(labels, n));
    *size = b.size();
    if (b.size() > cap) mgrx::fail(mgrx::errc::invalid_input, "capacity");
    std::memcpy(out, b.data(), b.size());
  });
}

int ref_lorenzo_f32(int nd, const uint64_t* dims, const float* data, double e, int32_t* labels, uint64_t* opos,
                    float* oval, uint64_t cap, uint64_t* n_out) {
  return lorenzo_t<float>(nd, dims, data, e, labels, opos, oval, cap, n_out);
}
int ref_lorenzo_f64(int nd, const uint64_t* dims, const double* data, double e, int32_t* labels, uint64_t* opos,
                    double* oval, uint64_t cap, uint64_t* n_out) {
  return lorenzo_t<double>(nd, dims, data, e, labels, opos, oval, cap, n_out);
}

int ref_choose_stop_f32(int nd, const uint64_t* dims, const float* data, double e, const double* interp_pen,
                        double lorenzo_pen, int step, double* totals, int* stop) {
  return choose_stop_t<float>(nd, dims, data, e, interp_pen, lorenzo_pen, step, totals, stop);
}
int ref_choose_stop_f64(int nd, const uint64_t* dims, const double* data, double e, const double* interp_pen,
                        double lorenzo_pen, int step, double* totals, int* stop) {
  return choose_stop_t<double>(nd, dims, data, e, interp_pen, lorenzo_pen, step, totals, stop);
}

const char* ref_last_error() { return g_msg; }

int ref_hierarchy(int nd, const uint64_t* dims, int levels, int* out_levels, uint64_t* level_dims,
                  uint64_t* delta_counts) {
  return guarded([&] {
    mgrx::GridHierarchy h = hier(nd, dims, levels);
    *out_levels = h.num_levels();
    if (level_dims)
      for (int l = 0; l <= h.num_levels(); ++l)
        for (int i = 0; i < nd; ++i)
          level_dims[static_cast<std::size_t>(l) * static_cast<std::size_t>(nd) + static_cast<std::size_t>(i)] =
              h.level_dims(l)[static_cast<std::size_t>(i)];
    if (delta_counts)
      for (int l = 0; l <= h.num_levels(); ++l) delta_counts[l] = h.delta_count(l);
  });
}

int ref_make_plan(int mode, double budget, int nd, const uint64_t* dims, int levels, double* q) {
  return guarded([&] {
    mgrx::GridHierarchy h = hier(nd, dims, levels);
    mgrx::QuantizationPlan p =
        mgrx::make_plan(mode == 0 ? mgrx::QuantMode::uniform : mgrx::QuantMode::levelwise, budget, h);
    std::memcpy(q, p.bin_widths.data(), p.bin_widths.size() * sizeof(double));
  });
}

int ref_estimated_cost(int mode, double budget, int nd, const uint64_t* dims, int levels,
                       double range, double* out) {
  return guarded([&] {
    mgrx::GridHierarchy h = hier(nd, dims, levels);
    mgrx::QuantizationPlan p =
        mgrx::make_plan(mode == 0 ? mgrx::QuantMode::uniform : mgrx::QuantMode::levelwise, budget, h);
    *out = mgrx::estimated_cost(p, h, range);
  });
}

int ref_decompose_f32(int nd, const uint64_t* dims, int levels, int stop, const float* in, float* out,
                      int batch) {
  return decompose_t<float>(nd, dims, levels, stop, in, out, batch);
}
int ref_decompose_f64(int nd, const uint64_t* dims, int levels, int stop, const double* in,
                      double* out, int batch) {
  return decompose_t<double>(nd, dims, levels, stop, in, out, batch);
}
int ref_recompose_f32(int nd, const uint64_t* dims, int levels, int stop, const float* in, float* out) {
  return recompose_t<float>(nd, dims, levels, stop, in, out);
}
int ref_recompose_f64(int nd, const uint64_t* dims, int levels, int stop, const double* in,
                      double* out) {
  return recompose_t<double>(nd, dims, levels, stop, in, out);
}
int ref_strided_decompose_f64(int nd, const uint64_t* dims, int levels, int stop, const double* in,
                              double* out) {
  return strided_decompose_t<double>(nd, dims, levels, stop, in, out);
}
int ref_quantize_f32(int nd, const uint64_t* dims, int levels, int stop, const double* q,
                     const float* c, int32_t* labels, uint64_t* opos, float* oval, uint64_t cap,
                     uint64_t* n_out) {
  return quantize_t<float>(nd, dims, levels, stop, q, c, labels, opos, oval, cap, n_out);
}
int ref_quantize_f64(int nd, const uint64_t* dims, int levels, int stop, const double* q,
                     const double* c, int32_t* labels, uint64_t* opos, double* oval, uint64_t cap,
                     uint64_t* n_out) {
  return quantize_t<double>(nd, dims, levels, stop, q, c, labels, opos, oval, cap, n_out);
}
int ref_dequantize_f32(int nd, const uint64_t* dims, int levels, int stop, const double* q,
                       const int32_t* labels, const uint64_t* opos, const float* oval,
                       uint64_t n_out, float* c) {
  return dequantize_t<float>(nd, dims, levels, stop, q, labels, opos, oval, n_out, c);
}
int ref_dequantize_f64(int nd, const uint64_t* dims, int levels, int stop, const double* q,
                       const int32_t* labels, const uint64_t* opos, const double* oval,
                       uint64_t n_out, double* c) {
  return dequantize_t<double>(nd, dims, levels, stop, q, labels, opos, oval, n_out, c);
}
int ref_level_step_f64(int nd, const uint64_t* dims, int level, double* field, double* corr) {
  return level_step_t<double>(nd, dims, level, field, corr);
}
int ref_level_step_f32(int nd, const uint64_t* dims, int level, float* field, double* corr) {
  return level_step_t<float>(nd, dims, level, field, corr);
}

int ref_load_vector_1d(const double* line, uint64_t n, double* out) {
  return guarded([&] {
    mgrx::load_vector_1d(std::span<const double>(line, n), std::span<double>(out, (n + 1) / 2));
  });
}
int ref_solve_correction_1d(double* f, uint64_t m) {
  return guarded([&] { mgrx::solve_correction_1d(std::span<double>(f, m)); });
}
int ref_thomas_aux(uint64_t m, double* w, double* inv_d) {
  return guarded([&] {
    mgrx::ThomasAux a = mgrx::ThomasAux::build(m);
    std::memcpy(w, a.w.data(), m * sizeof(double));
    std::memcpy(inv_d, a.inv_d.data(), m * sizeof(double));
  });
}
// Full reorder of all levels L..1 followed by pack_level_centric; used for
// layout fixtures (reorder.hpp:131,162).
int ref_reorder_pack_f64(int nd, const uint64_t* dims, int stop, const double* in, double* out) {
  return guarded([&] {
    mgrx::GridHierarchy h = hier(nd, dims, -1);
    mgrx::TensorField<double> f(to_dims(nd, dims));
    std::memcpy(f.data.data(), in, f.size() * sizeof(double));
    for (int l = h.num_levels(); l > stop; --l) mgrx::reorder_level(f, h, l);
    std::vector<double> b = mgrx::pack_level_centric(f, h, stop);
    std::memcpy(out, b.data(), b.size() * sizeof(double));
  });
}

} // extern "C"
