// Integration test of include/mgrx_b200.hpp against the unmodified reference
// (compiled by `make -C oracle dropin`; run on a GPU box by
// tests/test_gpu_dropin.py).  Checks the drop-in calls against the
// reference's own decompose / recompose / quantize / compress / decompress
// and that errors come back as mgrx::Error with the reference's errc.
#include <cmath>
#include <cstdio>
#include <string>
#include <limits>
#include <random>

#include "mgrx/pipeline.hpp"
#include "mgrx_b200.hpp"

static int failures = 0;
#define EXPECT(cond, ...)                       \
  do {                                          \
    if (!(cond)) {                              \
      ++failures;                               \
      std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
      std::printf(__VA_ARGS__);                 \
      std::printf("\n");                        \
    }                                           \
  } while (0)

template <typename T>
mgrx::TensorField<T> bumps(const mgrx::Dims& dims, unsigned seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  mgrx::TensorField<T> f(dims);
  const int d = int(dims.size());
  double c[8][3], w[8], a[8];
  for (int b = 0; b < 8; ++b) {
    for (int i = 0; i < 3; ++i) c[b][i] = u(rng);
    w[b] = 0.05 + 0.15 * u(rng);
    a[b] = 2.0 * u(rng) - 1.0;
  }
  std::vector<size_t> idx(dims.size(), 0);
  for (size_t p = 0; p < f.size(); ++p) {
    double v = 0.0;
    for (int b = 0; b < 8; ++b) {
      double r2 = 0.0;
      for (int i = 0; i < d; ++i) {
        const double x = double(idx[i]) / double(dims[i] - 1) - c[b][i % 3];
        r2 += x * x;
      }
      v += a[b] * std::exp(-r2 / (2.0 * w[b] * w[b]));
    }
    f.data[p] = T(v + 1e-3 * (u(rng) - 0.5));
    for (int i = d - 1; i >= 0; --i) {
      if (++idx[size_t(i)] < dims[size_t(i)]) break;
      idx[size_t(i)] = 0;
    }
  }
  return f;
}

template <typename T>
// exact_bytes: the device-resident compress must produce the reference's
// artifact byte for byte.  Off only for the fp64 fused-path case, whose
// coefficients differ from the reference's at the 1e-16 level (different
// rounding of the reordered sweeps); there the artifact size must match.
void check_shape(const mgrx::Dims& dims, double tol, bool exact_bytes = true) {
  mgrx::b200::Workspace ws;
  auto f = bumps<T>(dims, 7);
  double lo = f.data[0], hi = f.data[0];
  for (T v : f.data) {
    lo = std::min(lo, double(v));
    hi = std::max(hi, double(v));
  }
  const double range = hi - lo;
  const auto h = mgrx::GridHierarchy::create(dims);
  mgrx::SolverWorkspace sws;
  for (int stop : {0, 1}) {
    auto ref = mgrx::decompose(f, h, stop, sws);
    auto gpu = mgrx::b200::decompose(f, h, stop, ws);
    double err = 0.0;
    for (size_t i = 0; i < ref.buffer.size(); ++i)
      err = std::max(err, std::fabs(double(ref.buffer[i]) - double(gpu.buffer[i])));
    EXPECT(err <= tol * range, "decompose stop %d err %g", stop, err / range);
    auto back = mgrx::b200::recompose(gpu, ws);
    auto rback = mgrx::recompose(ref, sws);
    double e2 = 0.0;
    for (size_t i = 0; i < f.size(); ++i) e2 = std::max(e2, std::fabs(double(back.data[i]) - double(rback.data[i])));
    EXPECT(e2 <= tol * range, "recompose stop %d err %g", stop, e2 / range);
  }
  // quantize / dequantize: bit-exact labels from identical coefficients
  auto ref = mgrx::decompose(f, h, 0, sws);
  const auto plan = mgrx::make_plan(mgrx::QuantMode::levelwise, 1e-3 * range / 2.0, h);
  auto ls_ref = mgrx::quantize(ref, plan);
  auto ls_gpu = mgrx::b200::quantize(ref, plan, ws);
  EXPECT(ls_ref.labels == ls_gpu.labels, "labels differ");
  EXPECT(ls_ref.outliers.size() == ls_gpu.outliers.size(), "outlier count differs");
  auto dq_ref = mgrx::dequantize(ls_ref, plan, h);
  auto dq_gpu = mgrx::b200::dequantize(ls_gpu, plan, h, ws);
  EXPECT(dq_ref.buffer == dq_gpu.buffer, "dequantize differs");
  // compress on the GPU, decompress with the reference (and vice versa)
  // budget = tau / C with C = 4: the reference's budget is not an L-inf
  // bound and C = 2 is exceeded on this field
  mgrx::CompressOptions opt;
  opt.budget = 1e-3 * range / 4.0;
  opt.adaptive = false;
  auto bytes = mgrx::b200::compress(f, opt, ws);
  auto any = mgrx::decompress(bytes);
  const auto& rf = std::get<mgrx::TensorField<T>>(any);
  double linf = 0.0;
  for (size_t i = 0; i < f.size(); ++i) linf = std::max(linf, std::fabs(double(rf.data[i]) - double(f.data[i])));
  EXPECT(linf <= 1e-3 * range, "GPU-compressed artifact: linf/tau %g", linf / (1e-3 * range));
  auto bytes_ref = mgrx::compress(f, opt);
  auto gf = mgrx::b200::decompress_field<T>(mgrx::read_artifact(bytes_ref), ws);
  double linf2 = 0.0;
  for (size_t i = 0; i < f.size(); ++i) linf2 = std::max(linf2, std::fabs(double(gf.data[i]) - double(f.data[i])));
  EXPECT(linf2 <= 1e-3 * range, "reference artifact via GPU: linf/tau %g", linf2 / (1e-3 * range));
  EXPECT(std::fabs(linf - linf2) <= 1e-5 * range, "GPU and reference reconstructions differ: %g vs %g", linf, linf2);
  // decompose_with: a decider stopping at level L - 1 (and one never
  // stopping) gives the reference's buffer and stop level
  const int L = h.num_levels();
  for (int want : {L - 1, -1}) {
    std::vector<int> seen_ref, seen_gpu;
    mgrx::StopDecider<T> dref = [&](int level, const mgrx::BlockView<const T>&) {
      seen_ref.push_back(level);
      return level == want;
    };
    mgrx::StopDecider<T> dgpu = [&](int level, const mgrx::BlockView<const T>& b) {
      seen_gpu.push_back(level);
      EXPECT(b.extents == h.level_dims(level), "decider block extents at level %d", level);
      return level == want;
    };
    auto rw = mgrx::decompose_with(f, h, sws, dref);
    auto gw = mgrx::b200::decompose_with(f, h, ws, dgpu);
    EXPECT(rw.stop_level == gw.stop_level, "decompose_with stop %d vs %d", rw.stop_level, gw.stop_level);
    EXPECT(seen_ref == seen_gpu, "decider call sequence differs");
    double ew = 0.0;
    for (size_t i = 0; i < rw.buffer.size(); ++i)
      ew = std::max(ew, std::fabs(double(rw.buffer[i]) - double(gw.buffer[i])));
    EXPECT(ew <= tol * range, "decompose_with (stop at %d) err %g", want, ew / range);
  }
  // decompose_adaptive (choose_stop evaluated on the GPU on device-resident
  // level blocks) against the reference's decompose_with + choose_stop
  for (double rel : {1e-1, 1e-2, 1e-3, 1e-5}) {
    const auto plan = mgrx::make_plan(mgrx::QuantMode::levelwise, rel * range, h);
    const int d = int(dims.size());
    std::vector<int> ref_levels;
    mgrx::StopDecider<T> rdec = [&](int level, const mgrx::BlockView<const T>& b) {
      const double e_l = plan.bin_widths[static_cast<size_t>(level)] / 2.0;
      const double kappa = plan.bin_widths[static_cast<size_t>(level)] / plan.bin_widths[static_cast<size_t>(level - 1)];
      return mgrx::choose_stop(b, e_l, mgrx::penalty_model_for(d, kappa, 0));
    };
    auto rw = mgrx::decompose_with(f, h, sws, rdec);
    auto gw = mgrx::b200::decompose_adaptive(f, h, plan, 0, ws);
    EXPECT(rw.stop_level == gw.stop_level, "decompose_adaptive stop %d vs reference %d (budget %g)", gw.stop_level,
           rw.stop_level, rel);
    double ea = 0.0;
    for (size_t i = 0; i < rw.buffer.size(); ++i)
      ea = std::max(ea, std::fabs(double(rw.buffer[i]) - double(gw.buffer[i])));
    EXPECT(ea <= tol * range, "decompose_adaptive err %g (budget %g)", ea / range, rel);
    std::printf("  adaptive budget %g: stop %d\n", rel, gw.stop_level);
  }
  {  // check_finite (pipeline.hpp:132) on the GPU (fused into the finest
     // level's plane pass on the fused path): the reference's error code and
     // message (first non-finite offset), full and adaptive compress, NaN and inf
    for (int variant = 0; variant < 4; ++variant) {
      mgrx::TensorField<T> bad = f;
      const size_t at = bad.size() / 3 + size_t(variant);
      bad.data[at] = (variant & 1) ? std::numeric_limits<T>::infinity() : std::numeric_limits<T>::quiet_NaN();
      bad.data[bad.size() - 1] = -std::numeric_limits<T>::infinity();  // a later one: the first offset wins
      mgrx::CompressOptions o2 = opt;
      o2.adaptive = variant >= 2;
      std::string gmsg, rmsg;
      bool threw = false, rthrew = false;
      try {
        mgrx::b200::compress(bad, o2, ws);
      } catch (const mgrx::Error& e) {
        threw = e.code() == mgrx::errc::nonfinite_data;
        gmsg = e.what();
      }
      try {
        mgrx::compress(bad, o2);
      } catch (const mgrx::Error& e) {
        rthrew = e.code() == mgrx::errc::nonfinite_data;
        rmsg = e.what();
      }
      EXPECT(threw && rthrew, "non-finite field (variant %d): expected nonfinite_data", variant);
      EXPECT(gmsg.find(std::to_string(at)) != std::string::npos, "message '%s' lacks offset %zu (reference: '%s')",
             gmsg.c_str(), at, rmsg.c_str());
    }
  }
  // adaptive compress (the reference's choose_stop decider) round trip
  mgrx::CompressOptions aopt;
  aopt.budget = 1e-3 * range / 4.0;
  aopt.adaptive = true;
  auto abytes = mgrx::b200::compress(f, aopt, ws);
  const auto ra = mgrx::read_artifact(abytes);
  const auto rr = mgrx::read_artifact(mgrx::compress(f, aopt));
  EXPECT(ra.stop_level == rr.stop_level, "adaptive stop %d vs reference %d", int(ra.stop_level), int(rr.stop_level));
  {  // the device-resident compress (GPU entropy coding) vs the reference's bytes
    const auto rbytes = mgrx::compress(f, aopt);
    std::printf("  adaptive artifact: %zu bytes (reference %zu)%s\n", abytes.size(), rbytes.size(),
                abytes == rbytes ? ", byte-identical" : "");
    if (exact_bytes)
      EXPECT(abytes == rbytes, "adaptive artifact differs from the reference's bytes");
    else
      EXPECT(abytes.size() == rbytes.size(), "adaptive artifact size %zu vs %zu", abytes.size(), rbytes.size());
    mgrx::CompressOptions fopt = aopt;
    fopt.adaptive = false;
    const auto gb = mgrx::b200::compress(f, fopt, ws), rb = mgrx::compress(f, fopt);
    std::printf("  full artifact: %zu bytes (reference %zu)%s\n", gb.size(), rb.size(),
                gb == rb ? ", byte-identical" : "");
    if (exact_bytes)
      EXPECT(gb == rb, "full artifact differs from the reference's bytes");
    else
      EXPECT(gb.size() == rb.size(), "full artifact size %zu vs %zu", gb.size(), rb.size());
    const auto fany = mgrx::decompress(gb);
    const auto& ff = std::get<mgrx::TensorField<T>>(fany);
    double fl = 0.0;
    for (size_t i = 0; i < f.size(); ++i) fl = std::max(fl, std::fabs(double(ff.data[i]) - double(f.data[i])));
    EXPECT(fl <= 1e-3 * range, "full GPU artifact: linf/tau %g", fl / (1e-3 * range));
  }
  const auto aany = mgrx::decompress(abytes);
  const auto& af = std::get<mgrx::TensorField<T>>(aany);
  double alinf = 0.0;
  for (size_t i = 0; i < f.size(); ++i) alinf = std::max(alinf, std::fabs(double(af.data[i]) - double(f.data[i])));
  EXPECT(alinf <= 1e-3 * range, "adaptive GPU artifact: linf/tau %g", alinf / (1e-3 * range));
  std::printf("shape ok: %zu dims, range %g, linf/tau %g, adaptive stop %d\n", dims.size(), range,
              linf / (1e-3 * range), int(ra.stop_level));
}

int main() {
  check_shape<double>({33, 33, 33}, 1e-12, /*exact_bytes=*/false);
  check_shape<float>({65, 65, 65}, 1e-5);
  check_shape<float>({40, 36, 66}, 1e-5);
  check_shape<double>({17, 12}, 1e-12);
  check_shape<float>({5, 5, 5, 5}, 1e-5);
  // errors keep the reference's errc
  mgrx::b200::Workspace ws;
  const auto h = mgrx::GridHierarchy::create({9, 9});
  try {
    mgrx::b200::decompose(mgrx::TensorField<double>({9, 8}), h, 0, ws);
    EXPECT(false, "no throw");
  } catch (const mgrx::Error& e) {
    EXPECT(e.code() == mgrx::errc::shape_error, "errc %d", int(e.code()));
  }
  try {
    mgrx::b200::decompose(mgrx::TensorField<double>({9, 9}), h, 7, ws);
    EXPECT(false, "no throw");
  } catch (const mgrx::Error& e) {
    EXPECT(e.code() == mgrx::errc::invalid_level, "errc %d", int(e.code()));
  }
  mgrx::MultilevelCoefficients<double> bad{std::vector<double>(h.total_count(), 0.0), h, 0};
  bad.buffer[3] = NAN;
  try {
    mgrx::b200::quantize(bad, mgrx::make_plan(mgrx::QuantMode::uniform, 0.1, h), ws);
    EXPECT(false, "no throw");
  } catch (const mgrx::Error& e) {
    EXPECT(e.code() == mgrx::errc::nonfinite_data, "errc %d", int(e.code()));
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "ALL OK", failures);
  return failures ? 1 : 0;
}
