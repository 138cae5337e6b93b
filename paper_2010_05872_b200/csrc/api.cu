// C-ABI layer of mgrx_b200 (include/mgrx_b200.h): contexts, launch plans,
// scratch management and the level loops of decompose / recompose
// (reference transform.hpp:485-530) and quantize / dequantize
// (quantize.hpp:79-150).  Host-side only; all arithmetic runs in the
// kernels of general.cu, fused3d.cu and quantize.cu.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <queue>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "fused2d.h"
#include "fused3d.h"
#include "kernels.h"

using namespace mgrx_b200;

namespace {

// ---------------------------------------------------------------- errors

struct Status {
  int code = MGRX_OK;
  std::string msg;
};

struct Fail {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  throw Fail{code, buf};
}

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  const int code = (e == cudaErrorMemoryAllocation) ? MGRX_OUT_OF_MEMORY : MGRX_CUDA_ERROR;
  fail(code, "%s: %s", what, cudaGetErrorString(e));
}

// ------------------------------------------------------------- hierarchy
// GridHierarchy::max_levels / create (grid.cpp:9-49).

struct Hierarchy {
  int d = 0, L = 0;
  std::vector<std::vector<int64_t>> dims;  // [level][axis], level 0 coarsest
  std::vector<int64_t> node, delta;        // node_count / delta_count by level
};

int max_levels(int nd, const uint64_t* dims) {
  if (nd <= 0) fail(MGRX_INVALID_DIMS, "empty dimension list");
  if (nd > kMaxD) fail(MGRX_INVALID_DIMS, "rank %d exceeds %d", nd, kMaxD);
  int depth = 1 << 30;
  for (int i = 0; i < nd; ++i) {
    if (dims[i] < 2) fail(MGRX_INVALID_DIMS, "dimension %llu < 2", (unsigned long long)dims[i]);
    int k = 63 - __builtin_clzll(dims[i] - 1);  // floor(log2(n-1))
    depth = k < depth ? k : depth;
  }
  return depth;
}

Hierarchy make_hierarchy(int nd, const uint64_t* dims, int levels) {
  const int feasible = max_levels(nd, dims);
  const int L = levels < 0 ? feasible : levels;
  if (L > feasible) fail(MGRX_DEPTH_EXCEEDED, "requested %d levels, at most %d feasible", L, feasible);
  if (L + 1 > kMaxLevels) fail(MGRX_DEPTH_EXCEEDED, "too many levels");
  Hierarchy h;
  h.d = nd;
  h.L = L;
  h.dims.assign(L + 1, std::vector<int64_t>(nd));
  for (int i = 0; i < nd; ++i) h.dims[L][i] = int64_t(dims[i]);
  for (int l = L - 1; l >= 0; --l)
    for (int i = 0; i < nd; ++i) h.dims[l][i] = (h.dims[l + 1][i] + 1) / 2;
  h.node.resize(L + 1);
  h.delta.resize(L + 1);
  for (int l = 0; l <= L; ++l) {
    int64_t c = 1;
    for (int i = 0; i < nd; ++i) c *= h.dims[l][i];
    h.node[l] = c;
    h.delta[l] = c - (l ? h.node[l - 1] : 0);
  }
  return h;
}

LevelGeom make_geom(const Hierarchy& h, int l) {
  LevelGeom g{};
  g.d = h.d;
  for (int i = 0; i < h.d; ++i) {
    g.n[i] = h.dims[l][i];
    g.m[i] = h.dims[l - 1][i];
  }
  g.st[h.d - 1] = 1;
  g.cst[h.d - 1] = 1;
  for (int i = h.d - 2; i >= 0; --i) {
    g.st[i] = g.st[i + 1] * g.n[i + 1];
    g.cst[i] = g.cst[i + 1] * g.m[i + 1];
  }
  for (int i = 0; i < h.d; ++i) {
    int64_t p = 1;
    for (int k = i + 1; k + 1 < h.d; ++k) p *= g.m[k];
    g.pm[i] = p;
    g.fn[i] = FastDiv(uint32_t(g.n[i] <= 0xffffffffLL ? g.n[i] : 1));
  }
  g.N = h.node[l];
  g.Nc = h.node[l - 1];
  return g;
}

// ThomasAux::build (transform.hpp:29-43), identical constant expressions.
void thomas_aux(int64_t m, double* w, double* inv_d) {
  if (m < 2) fail(MGRX_DEGENERATE_SYSTEM, "correction system needs at least 2 unknowns");
  double dd = kDiagB;
  w[0] = 0.0;
  inv_d[0] = 1.0 / dd;
  for (int64_t i = 1; i < m; ++i) {
    const double wi = kOff / dd;
    w[i] = wi;
    dd = (i + 1 == m ? kDiagB : kDiagI) - wi * kOff;
    inv_d[i] = 1.0 / dd;
  }
}

// End-correction tables of the Toeplitz solves (fused3d.cu "Toeplitz
// solves"): with the constant factors w' = kTw, 1/d' = kTid the matrix
// T' = L' U' equals the correction matrix T except T'(0,0) = d' (T: 2/3) and
// T'(m-1,m-1) = w'/3 + d' (T: 2/3), so T = T' - a e_0 e_0^T - b e_l e_l^T and
// x = z + z_0 Gt + z_{m-1} Ht with z = T'^-1 f, Gt = a g / (1 - a g_0),
// Ht = b h / (1 - b h_{m-1}), g = T'^-1 e_0, h = T'^-1 e_{m-1} (the two ends
// decouple for m >= kToepMinM).  out: Gt[0..32) from the first row on,
// Ht[0..32) from the last row backwards.  Extended precision on the host.
void toeplitz_end_tables(int64_t m, double* out) {
  typedef long double ld;
  const ld w = ld(kTw), id = ld(kTid), d = 1.0L / id, o = ld(kOff);
  const ld a = d - ld(kDiagB), b = w * o + d - ld(kDiagB);
  const int64_t n = std::max<int64_t>(m, 2);
  std::vector<ld> y(n), g(n), h(n);
  y[0] = 1.0L;
  for (int64_t i = 1; i < n; ++i) y[i] = -w * y[i - 1];
  g[n - 1] = y[n - 1] * id;
  for (int64_t i = n - 2; i >= 0; --i) g[i] = (y[i] - o * g[i + 1]) * id;
  h[n - 1] = id;
  for (int64_t i = n - 2; i >= 0; --i) h[i] = -o * id * h[i + 1];
  const ld ca = a / (1.0L - a * g[0]), cb = b / (1.0L - b * h[n - 1]);
  for (int k = 0; k < kToepEnds; ++k) {
    out[k] = k < n ? double(ca * g[k]) : 0.0;
    out[kToepEnds + k] = k < n ? double(cb * h[n - 1 - k]) : 0.0;
  }
}

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// ------------------------------------------------------------------ plan

struct PlanKey {
  int dtype, L, stop;
  std::vector<int64_t> dims;
  bool operator<(const PlanKey& o) const {
    if (dtype != o.dtype) return dtype < o.dtype;
    if (L != o.L) return L < o.L;
    if (stop != o.stop) return stop < o.stop;
    return dims < o.dims;
  }
};

struct Plan {
  Hierarchy h;
  int stop = 0;
  size_t esize = 4;
  std::vector<LevelGeom> geom;     // index l (valid for l in (stop, L])
  std::vector<ThomasLevel> thomas; // index l
  double* d_tables = nullptr;      // uniform Thomas factors for all levels
  // scratch layout (bytes offsets)
  size_t off_comp = 0, off_tmp = 0, off_blk = 0, bytes = 0;
  std::vector<size_t> blk_off;     // level block offsets (levels stop..L-1)
  std::vector<Fused3DPlan> fused;  // index l; .enabled false when not applicable
  std::vector<Fused2DPlan> f2;     // index l; fused 2-D passes of nonuniform-coordinate calls
  // tail: levels stop+1..tail_top run in one CTA (uniform or nonuniform coordinates)
  int tail_top = -1;
  int64_t tail_nmax = 0;
  void* d_tail_dec = nullptr;  // TailLevel[] finest first
  void* d_tail_rec = nullptr;  // TailLevel[] coarsest first
  ~Plan() {
    if (d_tables) cudaFree(d_tables);
    if (d_tail_dec) cudaFree(d_tail_dec);
    if (d_tail_rec) cudaFree(d_tail_rec);
  }
};

}  // namespace

// Event profiler behind MGRX_LAUNCH (common.cuh): one start/stop event pair
// per tagged launch, recorded on the launching stream; summed per tag at
// mgrx_gpu_profile_end.
struct mgrx_b200::Profiler {
  struct Rec {
    const char* tag;
    int level;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  cudaEvent_t get() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  ~Profiler() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

void mgrx_b200::prof_mark(const Exec& ex, const char* tag, bool begin) {
  Profiler* p = ex.prof;
  if (begin) {
    cudaEvent_t a = p->get();
    cudaEventRecord(a, ex.s);
    p->recs.push_back({tag, ex.level, a, nullptr});
  } else {
    cudaEvent_t b = p->get();
    cudaEventRecord(b, ex.s);
    p->recs.back().b = b;
  }
}

struct mgrx_gpu_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  std::string last_error;
  uint64_t launches = 0;
  int path = 0;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  void* io = nullptr;  // host-entry-point staging (input + output)
  size_t io_bytes = 0;
  void* qtmp = nullptr;  // quantize chunk counts / offsets / flags
  size_t qtmp_bytes = 0;
  void* pinned = nullptr;  // pinned host readback
  double* nu_tables = nullptr;  // nonuniform per-call tables (device)
  uint64_t nu_key = 0;          // hash of (plan, coordinates) the tables were built for
  const void* nu_plan = nullptr;
  std::vector<NuLevel> nu_levels;
  NuLevel* d_tail_nu = nullptr;  // NuLevel of the tail levels: [dec order | rec order]
  size_t tail_nu_bytes = 0;
  size_t nu_bytes = 0;
  std::map<PlanKey, std::unique_ptr<Plan>> plans;
  Profiler prof;
  bool profiling = false;
  // recompose: side streams for the levels' independent corrections
  static constexpr int kSide = 4;
  cudaStream_t side[kSide] = {};
  cudaStream_t chain = nullptr;  // high priority: the sequential recompose chain
  cudaStream_t hi = nullptr;     // high priority: the finest level's correction (the critical path)
  cudaStream_t chain_lo = nullptr;  // low priority variant of the chain (MGRX_REC_PRIO=2)
  cudaEvent_t fork = nullptr, join = nullptr;
  std::vector<cudaEvent_t> lvl_done;
  // adaptive stop decision: per-block sums (device) and their host copy
  double* stop_dev = nullptr;
  size_t stop_dev_bytes = 0;
  // check_finite fused into the first decompose pass (compress): while
  // nf_armed, the next level decomposed on the fused 3-D path checks its
  // input into nf_flag and sets nf_used
  unsigned* nf_flag = nullptr;
  bool nf_armed = false, nf_used = false;
  double* stop_host = nullptr;
  size_t stop_host_bytes = 0;
  // dequantize + recompose: enqueued on the stream of the finest level's
  // correction before it (the finest shell's dequantization)
  std::function<void(cudaStream_t)> rec_pre_finest;
};

namespace {

Exec exec(mgrx_gpu_ctx* c, int level = -1) {
  return Exec{c->stream, &c->launches, c->profiling ? &c->prof : nullptr, level};
}

Exec exec_on(mgrx_gpu_ctx* c, cudaStream_t s, int level) {
  return Exec{s, &c->launches, c->profiling ? &c->prof : nullptr, level};
}

void ensure_side(mgrx_gpu_ctx* c, int levels) {
  if (!c->fork) {
    int least = 0, greatest = 0;
    cuda_check(cudaDeviceGetStreamPriorityRange(&least, &greatest), "cudaDeviceGetStreamPriorityRange");
    for (int i = 0; i < mgrx_gpu_ctx::kSide; ++i)
      cuda_check(cudaStreamCreateWithPriority(&c->side[i], cudaStreamNonBlocking, least), "cudaStreamCreate(side)");
    cuda_check(cudaStreamCreateWithPriority(&c->chain, cudaStreamNonBlocking, greatest), "cudaStreamCreate(chain)");
    cuda_check(cudaStreamCreateWithPriority(&c->hi, cudaStreamNonBlocking, greatest), "cudaStreamCreate(hi)");
    cuda_check(cudaStreamCreateWithPriority(&c->chain_lo, cudaStreamNonBlocking, least), "cudaStreamCreate(chain lo)");
    cuda_check(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming), "cudaEventCreate");
  }
  while (int(c->lvl_done.size()) < levels) {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    c->lvl_done.push_back(e);
  }
}

// Recompose stream priorities (MGRX_REC_PRIO, default 1): 0 = the chain high, every
// correction low; 1 = also the finest level's correction high; 2 = that
// correction high, the chain low.  (513^3, after the solves were reworked:
// 0.609 / 0.605 / 0.617 ms for 0 / 1 / 2.)
int rec_prio() {
  static const int v = std::getenv("MGRX_REC_PRIO") ? std::atoi(std::getenv("MGRX_REC_PRIO")) : 1;
  return v;
}

void set_device(mgrx_gpu_ctx* c) { cuda_check(cudaSetDevice(c->device), "cudaSetDevice"); }

void ensure(void** p, size_t* have, size_t need, mgrx_gpu_ctx* c, const char* what) {
  if (*have >= need) return;
  if (*p) {
    cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    cudaFree(*p);
    *p = nullptr;
    *have = 0;
  }
  cuda_check(cudaMalloc(p, need), what);
  *have = need;
}

size_t esize_of(int dtype) {
  if (dtype == MGRX_F32) return 4;
  if (dtype == MGRX_F64) return 8;
  fail(MGRX_INVALID_ARGUMENT, "unknown dtype %d", dtype);
}

Plan* get_plan(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int stop) {
  const size_t es = esize_of(dtype);
  Hierarchy h = make_hierarchy(nd, dims, levels);
  if (stop < 0 || stop > h.L) fail(MGRX_INVALID_LEVEL, "stop level %d out of range [0, %d]", stop, h.L);
  PlanKey key{dtype, h.L, stop, h.dims[h.L]};
  auto it = c->plans.find(key);
  if (it != c->plans.end()) return it->second.get();

  auto p = std::make_unique<Plan>();
  p->h = h;
  p->stop = stop;
  p->esize = es;
  const int L = h.L;
  p->geom.resize(L + 1);
  p->thomas.resize(L + 1);
  p->fused.resize(L + 1);
  // Uniform Thomas tables per level and axis (SolverWorkspace::prepare,
  // transform.hpp:58-61), uploaded once.
  std::vector<double> host;
  std::vector<std::pair<int, int>> slot;  // (level, axis) -> table starts
  std::vector<size_t> starts;
  for (int l = stop + 1; l <= L; ++l) {
    p->geom[l] = make_geom(h, l);
    for (int a = 0; a < nd; ++a) {
      const int64_t m = h.dims[l - 1][a];
      starts.push_back(host.size());
      host.resize(host.size() + 2 * size_t(m) + 2 * kToepEnds);  // w | inv_d | Toeplitz end corrections
      thomas_aux(m, host.data() + starts.back(), host.data() + starts.back() + m);
      toeplitz_end_tables(m, host.data() + starts.back() + 2 * m);
    }
  }
  if (!host.empty()) {
    cuda_check(cudaMalloc(&p->d_tables, host.size() * sizeof(double)), "cudaMalloc(tables)");
    cuda_check(cudaMemcpy(p->d_tables, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice),
               "upload tables");
  }
  size_t k = 0;
  for (int l = stop + 1; l <= L; ++l)
    for (int a = 0; a < nd; ++a, ++k) {
      const int64_t m = h.dims[l - 1][a];
      p->thomas[l].w[a] = p->d_tables + starts[k];
      p->thomas[l].inv_d[a] = p->d_tables + starts[k] + m;
    }
  // Tail: the small levels (block fits one CTA's shared memory) in one launch.
  {
    const int64_t tail_max = int64_t((220 * 1024) / (16 + 2 * es));
    int top = -1;
    for (int l = stop + 1; l <= L; ++l)
      if (h.node[l] <= tail_max) top = l;
    if (top > stop) {
      p->tail_top = top;
      p->tail_nmax = h.node[top];
      const int nlev = top - stop;
      const size_t lb = tail_level_bytes();
      std::vector<unsigned char> dec(nlev * lb), rec(nlev * lb);
      for (int k = 0; k < nlev; ++k) {
        const int ld = top - k, lr = stop + 1 + k;
        tail_fill_level(dec.data() + k * lb, p->geom[ld], p->thomas[ld], h.node[ld - 1]);
        tail_fill_level(rec.data() + k * lb, p->geom[lr], p->thomas[lr], h.node[lr - 1]);
      }
      cuda_check(cudaMalloc(&p->d_tail_dec, dec.size()), "cudaMalloc(tail)");
      cuda_check(cudaMalloc(&p->d_tail_rec, rec.size()), "cudaMalloc(tail)");
      cuda_check(cudaMemcpy(p->d_tail_dec, dec.data(), dec.size(), cudaMemcpyHostToDevice), "upload tail");
      cuda_check(cudaMemcpy(p->d_tail_rec, rec.data(), rec.size(), cudaMemcpyHostToDevice), "upload tail");
    }
  }
  // Scratch: fp64 component + sweep ping-pong (sized for the finest level
  // processed) and the compact level blocks stop..L-1.
  int64_t comp = 0, tmp = 0;
  for (int l = stop + 1; l <= L; ++l) {
    comp = std::max(comp, h.node[l]);
    int64_t y0 = h.dims[l - 1][0];
    for (int i = 1; i < nd; ++i) y0 *= h.dims[l][i];
    tmp = std::max(tmp, y0);
  }
  size_t off = 0;
  p->off_comp = off;
  off = align_up(off + size_t(comp) * 8);
  p->off_tmp = off;
  off = align_up(off + size_t(tmp) * 8);
  p->blk_off.assign(L + 1, 0);
  for (int l = stop; l < L; ++l) {
    p->blk_off[l] = off;
    off = align_up(off + size_t(h.node[l]) * es);
  }
  // Fused 3-D plans (fused3d.cu) for the levels they cover.
  for (int l = stop + 1; l <= L; ++l) {
    p->fused[l] = fused3d_plan(p->geom[l], int(es));
    if (p->fused[l].enabled) {
      p->fused[l].scratch_off = off;
      off = align_up(off + p->fused[l].scratch_bytes);
    }
  }
  p->f2.resize(L + 1);
  for (int l = stop + 1; l <= L; ++l) {
    p->f2[l] = fused2d_plan(p->geom[l]);
    if (p->f2[l].enabled) {
      p->f2[l].scratch_off = off;
      off = align_up(off + p->f2[l].scratch_bytes);
    }
  }
  p->bytes = off;
  Plan* raw = p.get();
  c->plans.emplace(key, std::move(p));
  return raw;
}

// ----------------------------------------------------- nonuniform tables
// Same derivation as oracle/mgrx_oracle.c:nu_build (uniform spacing
// reduces every table to the reference constants).  Host fp64, uploaded per
// call into ctx->nu_tables.
void nu_axis_tables(const double* x, int64_t n, std::vector<double>& out, size_t* o_wl, size_t* o_wr,
                    size_t* o_s, size_t* o_tw, size_t* o_tid, size_t* o_off) {
  const int64_t m = (n + 1) / 2;
  *o_wl = out.size();
  out.resize(out.size() + n, 0.0);
  *o_wr = out.size();
  out.resize(out.size() + n, 0.0);
  *o_s = out.size();
  out.resize(out.size() + 5 * m, 0.0);
  *o_tw = out.size();
  out.resize(out.size() + m, 0.0);
  *o_tid = out.size();
  out.resize(out.size() + m, 0.0);
  *o_off = out.size();
  out.resize(out.size() + m, 0.0);
  double* wl = out.data() + *o_wl;
  double* wr = out.data() + *o_wr;
  double* s = out.data() + *o_s;
  double* tw = out.data() + *o_tw;
  double* tid = out.data() + *o_tid;
  double* offd = out.data() + *o_off;
  for (int64_t j = 1; j < n; j += 2) {
    if (j + 1 < n) {
      const double span = x[j + 1] - x[j - 1];
      wl[j] = (x[j + 1] - x[j]) / span;
      wr[j] = (x[j] - x[j - 1]) / span;
    } else {
      wl[j] = 1.0;
      wr[j] = 0.0;
    }
  }
  auto H = [&](int64_t j) { return (j >= 0 && j + 1 < n) ? x[j + 1] - x[j] : 0.0; };
  for (int64_t i = 0; i < m; ++i) {
    const int64_t c = 2 * i;
    double* si = s + 5 * i;
    const bool even_end = (n % 2 == 0) && (i + 1 == m);
    const double al = i > 0 ? H(c - 2) / (H(c - 2) + H(c - 1)) : 0.0;
    const double ar = (!even_end && i + 1 < m) ? H(c + 1) / (H(c) + H(c + 1)) : 0.0;
    if (i > 0) {
      si[0] = al * H(c - 2) / 6.0;
      si[1] = al * (H(c - 2) + H(c - 1)) / 3.0 + H(c - 1) / 6.0;
    }
    if (even_end) {
      si[2] = al * H(c - 1) / 6.0 + H(c - 1) / 3.0;
      si[3] = H(c) / 2.0;
    } else {
      si[2] = al * H(c - 1) / 6.0 + (H(c - 1) + H(c)) / 3.0 + ar * H(c) / 6.0;
      if (i + 1 < m) {
        si[3] = H(c) / 6.0 + ar * (H(c) + H(c + 1)) / 3.0;
        si[4] = ar * H(c + 1) / 6.0;
      }
    }
  }
  std::vector<double> Hc(m, 0.0);
  for (int64_t i = 0; i + 1 < m; ++i) Hc[i] = x[2 * i + 2] - x[2 * i];
  double dd = Hc[0] / 3.0;
  tw[0] = 0.0;
  tid[0] = 1.0 / dd;
  for (int64_t i = 0; i + 1 < m; ++i) offd[i] = Hc[i] / 6.0;
  for (int64_t i = 1; i < m; ++i) {
    const double wi = offd[i - 1] / dd;
    tw[i] = wi;
    const double diag = (Hc[i - 1] + (i + 1 < m ? Hc[i] : 0.0)) / 3.0;
    dd = diag - wi * offd[i - 1];
    tid[i] = 1.0 / dd;
  }
}

std::vector<NuLevel> upload_nu(mgrx_gpu_ctx* c, const Plan& p, const double* const* coords) {
  const Hierarchy& h = p.h;
  if (!coords) fail(MGRX_INVALID_ARGUMENT, "coords is NULL");
  uint64_t key = 1469598103934665603ull;  // FNV-1a over the coordinates
  for (int a = 0; a < h.d; ++a) {
    if (!coords[a]) fail(MGRX_INVALID_ARGUMENT, "coords[%d] is NULL", a);
    for (int64_t j = 0; j + 1 < h.dims[h.L][a]; ++j)
      if (!(coords[a][j + 1] > coords[a][j]))
        fail(MGRX_INVALID_INPUT, "coordinates of axis %d not strictly increasing at %lld", a, (long long)j);
    const unsigned char* b = reinterpret_cast<const unsigned char*>(coords[a]);
    for (size_t i = 0; i < size_t(h.dims[h.L][a]) * sizeof(double); ++i) key = (key ^ b[i]) * 1099511628211ull;
  }
  // same plan and coordinates as the last call: the device tables are
  // current (no upload, so the call can be captured in a CUDA graph)
  if (c->nu_plan == &p && c->nu_key == key && !c->nu_levels.empty()) return c->nu_levels;
  std::vector<double> host;
  struct Off {
    size_t wl, wr, s, tw, tid, off;
  };
  std::vector<std::vector<Off>> offs(h.L + 1, std::vector<Off>(h.d));
  std::vector<double> x;
  for (int l = p.stop + 1; l <= h.L; ++l)
    for (int a = 0; a < h.d; ++a) {
      const int64_t n = h.dims[l][a];
      const int64_t stride = int64_t(1) << (h.L - l);
      x.resize(n);
      for (int64_t j = 0; j < n; ++j) x[j] = coords[a][j * stride];
      Off& o = offs[l][a];
      nu_axis_tables(x.data(), n, host, &o.wl, &o.wr, &o.s, &o.tw, &o.tid, &o.off);
    }
  size_t need = host.size() * sizeof(double);
  ensure(reinterpret_cast<void**>(&c->nu_tables), &c->nu_bytes, need ? need : 8, c, "cudaMalloc(nu tables)");
  cuda_check(cudaMemcpyAsync(c->nu_tables, host.data(), need, cudaMemcpyHostToDevice, c->stream), "upload nu");
  std::vector<NuLevel> out(h.L + 1);
  for (int l = p.stop + 1; l <= h.L; ++l)
    for (int a = 0; a < h.d; ++a) {
      const Off& o = offs[l][a];
      out[l].ax[a] = NuAxis{c->nu_tables + o.wl, c->nu_tables + o.wr, c->nu_tables + o.s,
                            c->nu_tables + o.tw, c->nu_tables + o.tid, c->nu_tables + o.off};
    }
  // the tail kernels' per-level tables, in their level orders
  std::vector<NuLevel> tail;
  if (p.tail_top > p.stop) {
    for (int l = p.tail_top; l > p.stop; --l) tail.push_back(out[l]);   // decompose: finest first
    for (int l = p.stop + 1; l <= p.tail_top; ++l) tail.push_back(out[l]);  // recompose: coarsest first
    ensure(reinterpret_cast<void**>(&c->d_tail_nu), &c->tail_nu_bytes, tail.size() * sizeof(NuLevel), c,
           "cudaMalloc(tail nu)");
    cuda_check(cudaMemcpyAsync(c->d_tail_nu, tail.data(), tail.size() * sizeof(NuLevel), cudaMemcpyHostToDevice,
                               c->stream),
               "upload tail nu");
  }
  cuda_check(cudaStreamSynchronize(c->stream), "sync nu upload");
  c->nu_plan = &p;
  c->nu_key = key;
  c->nu_levels = out;
  return out;
}

// ------------------------------------------------------------- transform

// finest_shell_done: when given and the finest level runs on the fused 3-D
// path, the event is recorded right after that level's plane pass (its shell
// is final from then on) and *shell_event_used is set.
template <typename T>
void decompose_impl(mgrx_gpu_ctx* c, Plan& p, const T* d_field, T* d_out, const std::vector<NuLevel>* nu,
                    cudaEvent_t finest_shell_done = nullptr, bool* shell_event_used = nullptr) {
  const Hierarchy& h = p.h;
  const int L = h.L, stop = p.stop;
  if (stop == L) {  // identity (transform.hpp:494 loop does not run)
    cuda_check(cudaMemcpyAsync(d_out, d_field, size_t(h.node[L]) * sizeof(T), cudaMemcpyDeviceToDevice, c->stream),
               "copy");
    return;
  }
  ensure(&c->scratch, &c->scratch_bytes, p.bytes, c, "cudaMalloc(scratch)");
  char* s = static_cast<char*>(c->scratch);
  double* comp = reinterpret_cast<double*>(s + p.off_comp);
  double* tmp = reinterpret_cast<double*>(s + p.off_tmp);
  const T* blk = d_field;
  const bool nf_arm = c->nf_armed;  // only this call's finest level can carry the check
  c->nf_armed = false;
  for (int l = L; l > stop; --l) {
    if (l == p.tail_top) {  // levels l..stop+1 in one CTA
      cuda_check(tail_decompose<T>(blk, d_out, d_out, p.d_tail_dec, nu ? c->d_tail_nu : nullptr, l - stop,
                                   p.tail_nmax, h.d, exec(c, l)),
                 "tail");
      break;
    }
    T* shell = d_out + h.node[l - 1];
    T* coarse = (l - 1 == stop) ? d_out : reinterpret_cast<T*>(s + p.blk_off[l - 1]);
    const Fused3DPlan& fp = p.fused[l];
    cudaError_t e;
    if (nu && c->path == 0 && p.f2[l].enabled) {
      e = fused2d_decompose_level<T>(blk, shell, coarse, s + p.f2[l].scratch_off, p.f2[l], (*nu)[l], exec(c, l));
    } else if (!nu && c->path == 0 && fp.enabled) {
      Exec ex = exec(c, l);
      if (nf_arm && l == L) {  // check_finite rides on this level's plane pass
        ex.nonfinite = c->nf_flag;
        c->nf_used = true;
      }
      if (finest_shell_done && l == L) {
        ex.after_plane = finest_shell_done;
        if (shell_event_used) *shell_event_used = true;
      }
      e = fused3d_decompose_level<T>(blk, shell, coarse, s + fp.scratch_off, p.geom[l], fp, p.thomas[l], ex);
    } else {
      e = general_decompose_level<T>(blk, shell, coarse, comp, tmp, p.geom[l], &p.thomas[l],
                                     nu ? &(*nu)[l] : nullptr, exec(c, l), c->path == 0);
    }
    cuda_check(e, "decompose level");
    blk = coarse;
  }
}

template <typename T>
void recompose_impl(mgrx_gpu_ctx* c, Plan& p, const T* d_coeffs, T* d_field, const std::vector<NuLevel>* nu) {
  const Hierarchy& h = p.h;
  const int L = h.L, stop = p.stop;
  if (stop == L) {
    cuda_check(cudaMemcpyAsync(d_field, d_coeffs, size_t(h.node[L]) * sizeof(T), cudaMemcpyDeviceToDevice,
                               c->stream),
               "copy");
    return;
  }
  ensure(&c->scratch, &c->scratch_bytes, p.bytes, c, "cudaMalloc(scratch)");
  char* s = static_cast<char*>(c->scratch);
  double* comp = reinterpret_cast<double*>(s + p.off_comp);
  double* tmp = reinterpret_cast<double*>(s + p.off_tmp);
  // Corrections of the fused levels depend only on their shells
  // (transform.hpp:343-366: the component is zero on the coarse nodes): fork
  // them onto side streams at the start; the sequential chain (tail, then per
  // level axis-0 solve + apply + interpolation) runs on a high-priority
  // stream, waiting for each level's correction; everything joins back into
  // the caller's stream.  Not while profiling (per-kernel event times need
  // the serial order).
  std::vector<char> forked(L + 1, 0);
  cudaStream_t cs = c->stream;  // the chain's stream
  {
    int nf = 0;
    if (!nu && c->path == 0 && !c->profiling)
      for (int l = stop + 1; l <= L; ++l) nf += p.fused[l].enabled ? 1 : 0;
    if (nf > 0) {
      ensure_side(c, L + 1);
      cuda_check(cudaEventRecord(c->fork, c->stream), "cudaEventRecord(fork)");
      int k = 0;
      // coarse levels first: their corrections are small and the chain needs
      // them first; the finest level's large correction is enqueued last
      for (int l = stop + 1; l <= L; ++l) {
        const Fused3DPlan& fp = p.fused[l];
        if (!fp.enabled) continue;
        cudaStream_t sd = c->side[k++ % mgrx_gpu_ctx::kSide];
        if (l == L && rec_prio() >= 1) sd = c->hi;
        cuda_check(cudaStreamWaitEvent(sd, c->fork, 0), "cudaStreamWaitEvent");
        if (l == L && c->rec_pre_finest) c->rec_pre_finest(sd);
        cuda_check(fused3d_recompose_correction<T>(d_coeffs + h.node[l - 1], s + fp.scratch_off, fp, p.thomas[l],
                                                   exec_on(c, sd, l)),
                   "recompose correction");
        cuda_check(cudaEventRecord(c->lvl_done[l], sd), "cudaEventRecord");
        forked[l] = 1;
      }
      cs = rec_prio() == 2 ? c->chain_lo : c->chain;
      cuda_check(cudaStreamWaitEvent(cs, c->fork, 0), "cudaStreamWaitEvent");
    }
  }
  // unpack_level_centric's coarse block (reorder.hpp:231-238)
  T* coarse = reinterpret_cast<T*>(s + p.blk_off[stop]);
  int l0 = stop + 1;
  if (p.tail_top > stop) {  // levels stop+1..tail_top in one CTA
    const int top = p.tail_top;
    T* fine = (top == L) ? d_field : reinterpret_cast<T*>(s + p.blk_off[top]);
    cuda_check(tail_recompose<T>(d_coeffs, d_coeffs, fine, p.d_tail_rec,
                                 nu ? static_cast<const void*>(c->d_tail_nu + (top - stop)) : nullptr, top - stop,
                                 p.tail_nmax, h.d,
                                    exec_on(c, cs, top)), "tail");
    coarse = fine;
    l0 = top + 1;
  } else {
    cuda_check(cudaMemcpyAsync(coarse, d_coeffs, size_t(h.node[stop]) * sizeof(T), cudaMemcpyDeviceToDevice, cs),
               "copy coarse");
  }
  for (int l = l0; l <= L; ++l) {
    const T* shell = d_coeffs + h.node[l - 1];
    T* fine = (l == L) ? d_field : reinterpret_cast<T*>(s + p.blk_off[l]);
    const Fused3DPlan& fp = p.fused[l];
    cudaError_t e;
    if (forked[l]) {
      cuda_check(cudaStreamWaitEvent(cs, c->lvl_done[l], 0), "cudaStreamWaitEvent");
      e = fused3d_recompose_finish<T>(shell, coarse, fine, s + fp.scratch_off, fp, p.thomas[l], exec_on(c, cs, l));
    } else if (nu && c->path == 0 && p.f2[l].enabled) {
      e = fused2d_recompose_level<T>(shell, coarse, fine, s + p.f2[l].scratch_off, p.f2[l], (*nu)[l],
                                     exec_on(c, cs, l));
    } else if (!nu && c->path == 0 && fp.enabled) {
      e = fused3d_recompose_level<T>(shell, coarse, fine, s + fp.scratch_off, p.geom[l], fp, p.thomas[l],
                                     exec_on(c, cs, l));
    } else {
      e = general_recompose_level<T>(shell, coarse, fine, comp, tmp, p.geom[l], &p.thomas[l],
                                     nu ? &(*nu)[l] : nullptr, exec_on(c, cs, l), c->path == 0);
    }
    cuda_check(e, "recompose level");
    coarse = fine;
  }
  if (cs != c->stream) {  // join the chain (which joined every side stream)
    cuda_check(cudaEventRecord(c->join, cs), "cudaEventRecord(join)");
    cuda_check(cudaStreamWaitEvent(c->stream, c->join, 0), "cudaStreamWaitEvent");
  }
}

QuantLevels quant_levels(const Plan& p, const double* q) {
  const Hierarchy& h = p.h;
  QuantLevels ql{};
  ql.first = p.stop == 0 ? 0 : p.stop + 1;
  ql.last = h.L;
  ql.base = p.stop == 0 ? 0 : h.node[p.stop];
  ql.total = h.node[h.L];
  for (int l = 0; l <= h.L; ++l) {
    ql.end[l] = h.node[l];
    ql.q[l] = q[l];
    ql.inv[l] = 1.0 / q[l];
  }
  return ql;
}

template <typename Fn>
int guarded(mgrx_gpu_ctx* c, Fn&& fn) {
  if (!c) return MGRX_INVALID_ARGUMENT;
  try {
    set_device(c);
    fn();
    return MGRX_OK;
  } catch (const Fail& f) {
    c->last_error = f.msg;
    return f.code;
  } catch (const std::bad_alloc&) {
    c->last_error = "host allocation failed";
    return MGRX_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    c->last_error = e.what();
    return MGRX_INVALID_ARGUMENT;
  }
}

template <typename Fn>
int guarded_noctx(Fn&& fn) {
  try {
    fn();
    return MGRX_OK;
  } catch (const Fail& f) {
    return f.code;
  } catch (...) {
    return MGRX_INVALID_ARGUMENT;
  }
}

}  // namespace

// =========================================================================
extern "C" {

int mgrx_abi_version(void) { return MGRX_B200_ABI_VERSION; }

int mgrx_gpu_ctx_create(int device, mgrx_gpu_ctx** out) {
  if (!out) return MGRX_INVALID_ARGUMENT;
  *out = nullptr;
  auto* c = new (std::nothrow) mgrx_gpu_ctx;
  if (!c) return MGRX_OUT_OF_MEMORY;
  c->device = device;
  int rc = guarded(c, [&] {
    cuda_check(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking), "cudaStreamCreate");
    c->stream = c->own;
    cuda_check(cudaMallocHost(&c->pinned, 64), "cudaMallocHost");
  });
  if (rc != MGRX_OK) {
    delete c;
    return rc;
  }
  *out = c;
  return MGRX_OK;
}

int mgrx_gpu_ctx_destroy(mgrx_gpu_ctx* c) {
  if (!c) return MGRX_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  c->plans.clear();
  if (c->scratch) cudaFree(c->scratch);
  if (c->io) cudaFree(c->io);
  if (c->qtmp) cudaFree(c->qtmp);
  if (c->nu_tables) cudaFree(c->nu_tables);
  if (c->d_tail_nu) cudaFree(c->d_tail_nu);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->own) cudaStreamDestroy(c->own);
  for (int i = 0; i < mgrx_gpu_ctx::kSide; ++i)
    if (c->side[i]) cudaStreamDestroy(c->side[i]);
  if (c->chain) cudaStreamDestroy(c->chain);
  if (c->hi) cudaStreamDestroy(c->hi);
  if (c->chain_lo) cudaStreamDestroy(c->chain_lo);
  if (c->fork) cudaEventDestroy(c->fork);
  if (c->join) cudaEventDestroy(c->join);
  for (cudaEvent_t e : c->lvl_done) cudaEventDestroy(e);
  if (c->stop_dev) cudaFree(c->stop_dev);
  if (c->nf_flag) cudaFree(c->nf_flag);
  if (c->stop_host) cudaFreeHost(c->stop_host);
  delete c;
  return MGRX_OK;
}

int mgrx_gpu_set_stream(mgrx_gpu_ctx* c, void* stream) {
  return guarded(c, [&] { c->stream = static_cast<cudaStream_t>(stream); });
}

void* mgrx_gpu_get_stream(mgrx_gpu_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int mgrx_gpu_synchronize(mgrx_gpu_ctx* c) {
  return guarded(c, [&] { cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize"); });
}

const char* mgrx_gpu_last_error(const mgrx_gpu_ctx* c) { return c ? c->last_error.c_str() : "null context"; }

uint64_t mgrx_gpu_launch_count(const mgrx_gpu_ctx* c) { return c ? c->launches : 0; }

int mgrx_gpu_profile_begin(mgrx_gpu_ctx* c) {
  return guarded(c, [&] {
    c->prof.recs.clear();
    c->prof.used = 0;
    c->profiling = true;
  });
}

int mgrx_gpu_profile_end(mgrx_gpu_ctx* c, char* tags, double* ms, uint64_t* counts, int cap, int* n) {
  return guarded(c, [&] {
    c->profiling = false;
    cuda_check(cudaStreamSynchronize(c->stream), "profile sync");
    std::vector<std::string> names;
    std::vector<double> tot;
    std::vector<uint64_t> cnt;
    for (const auto& r : c->prof.recs) {
      float t = 0.f;
      cuda_check(cudaEventElapsedTime(&t, r.a, r.b), "cudaEventElapsedTime");
      const std::string key = r.level >= 0 ? std::string(r.tag) + "@" + std::to_string(r.level) : std::string(r.tag);
      size_t i = 0;
      while (i < names.size() && names[i] != key) ++i;
      if (i == names.size()) {
        names.push_back(key);
        tot.push_back(0.0);
        cnt.push_back(0);
      }
      tot[i] += t;
      cnt[i] += 1;
    }
    *n = int(names.size());
    for (int i = 0; i < int(names.size()) && i < cap; ++i) {
      std::snprintf(tags + 32 * i, 32, "%s", names[i].c_str());
      ms[i] = tot[i];
      counts[i] = cnt[i];
    }
    c->prof.recs.clear();
    c->prof.used = 0;
  });
}

int mgrx_gpu_set_path(mgrx_gpu_ctx* c, int path) {
  return guarded(c, [&] {
    if (path < 0 || path > 1) fail(MGRX_INVALID_ARGUMENT, "path must be 0 (auto) or 1 (general)");
    c->path = path;
  });
}

int mgrx_hierarchy(int nd, const uint64_t* dims, int levels, int* out_levels, uint64_t* level_dims,
                   uint64_t* delta_counts) {
  return guarded_noctx([&] {
    if (!out_levels || (nd > 0 && !dims)) fail(MGRX_INVALID_ARGUMENT, "null argument");
    Hierarchy h = make_hierarchy(nd, dims, levels);
    *out_levels = h.L;
    for (int l = 0; l <= h.L; ++l) {
      if (level_dims)
        for (int i = 0; i < nd; ++i) level_dims[size_t(l) * nd + i] = uint64_t(h.dims[l][i]);
      if (delta_counts) delta_counts[l] = uint64_t(h.delta[l]);
    }
  });
}

int mgrx_make_plan(int mode, double budget, int nd, const uint64_t* dims, int levels, double* q) {
  return guarded_noctx([&] {
    if (!(budget > 0.0) || !std::isfinite(budget)) fail(MGRX_INVALID_BUDGET, "budget must be positive");
    if (!dims || !q) fail(MGRX_INVALID_ARGUMENT, "null argument");
    Hierarchy h = make_hierarchy(nd, dims, levels);
    const int L = h.L;
    if (mode == MGRX_QUANT_UNIFORM) {
      const double qq = 2.0 * budget / double(L + 1);
      for (int l = 0; l <= L; ++l) q[l] = qq;
    } else if (mode == MGRX_QUANT_LEVELWISE) {
      const double total = double(h.node[L]);
      for (int l = 0; l <= L; ++l) q[l] = 2.0 * budget * double(h.delta[l]) / total;
    } else {
      fail(MGRX_INVALID_ARGUMENT, "unknown quant mode %d", mode);
    }
  });
}

int mgrx_gpu_workspace_size(int dtype, int nd, const uint64_t* dims, int levels, int stop, uint64_t* bytes) {
  mgrx_gpu_ctx tmp;  // plan sizing only; no device work besides table upload
  int rc = guarded(&tmp, [&] {
    Plan* p = get_plan(&tmp, dtype, nd, dims, levels, stop);
    *bytes = p->bytes;
  });
  tmp.plans.clear();
  return rc;
}

int mgrx_gpu_decompose(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int stop,
                       const void* d_field, void* d_out) {
  return guarded(c, [&] {
    if (!dims || !d_field || !d_out) fail(MGRX_INVALID_ARGUMENT, "null argument");
    Plan* p = get_plan(c, dtype, nd, dims, levels, stop);
    if (dtype == MGRX_F32)
      decompose_impl<float>(c, *p, static_cast<const float*>(d_field), static_cast<float*>(d_out), nullptr);
    else
      decompose_impl<double>(c, *p, static_cast<const double*>(d_field), static_cast<double*>(d_out), nullptr);
  });
}

int mgrx_gpu_recompose(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int stop,
                       const void* d_coeffs, void* d_field) {
  return guarded(c, [&] {
    if (!dims || !d_coeffs || !d_field) fail(MGRX_INVALID_ARGUMENT, "null argument");
    Plan* p = get_plan(c, dtype, nd, dims, levels, stop);
    if (dtype == MGRX_F32)
      recompose_impl<float>(c, *p, static_cast<const float*>(d_coeffs), static_cast<float*>(d_field), nullptr);
    else
      recompose_impl<double>(c, *p, static_cast<const double*>(d_coeffs), static_cast<double*>(d_field), nullptr);
  });
}

int mgrx_gpu_decompose_nonuniform(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int stop,
                                  const double* const* coords, const void* d_field, void* d_out) {
  return guarded(c, [&] {
    if (!dims || !d_field || !d_out) fail(MGRX_INVALID_ARGUMENT, "null argument");
    Plan* p = get_plan(c, dtype, nd, dims, levels, stop);
    std::vector<NuLevel> nu = upload_nu(c, *p, coords);
    if (dtype == MGRX_F32)
      decompose_impl<float>(c, *p, static_cast<const float*>(d_field), static_cast<float*>(d_out), &nu);
    else
      decompose_impl<double>(c, *p, static_cast<const double*>(d_field), static_cast<double*>(d_out), &nu);
  });
}

int mgrx_gpu_recompose_nonuniform(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int stop,
                                  const double* const* coords, const void* d_coeffs, void* d_field) {
  return guarded(c, [&] {
    if (!dims || !d_coeffs || !d_field) fail(MGRX_INVALID_ARGUMENT, "null argument");
    Plan* p = get_plan(c, dtype, nd, dims, levels, stop);
    std::vector<NuLevel> nu = upload_nu(c, *p, coords);
    if (dtype == MGRX_F32)
      recompose_impl<float>(c, *p, static_cast<const float*>(d_coeffs), static_cast<float*>(d_field), &nu);
    else
      recompose_impl<double>(c, *p, static_cast<const double*>(d_coeffs), static_cast<double*>(d_field), &nu);
  });
}

int mgrx_gpu_quantize(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int stop,
                      const double* q, const void* d_coeffs, int32_t* d_labels, uint64_t* d_opos, void* d_oval,
                      uint64_t capacity, uint64_t* n_outliers) {
  return guarded(c, [&] {
    if (!dims || !q || !d_coeffs || !d_labels || !n_outliers) fail(MGRX_INVALID_ARGUMENT, "null argument");
    Plan* p = get_plan(c, dtype, nd, dims, levels, stop);
    for (int l = 0; l <= p->h.L; ++l)
      if (!(q[l] > 0.0) || !std::isfinite(q[l])) fail(MGRX_INVALID_BUDGET, "bad bin width at level %d", l);
    QuantLevels ql = quant_levels(*p, q);
    const int64_t nch = quant_num_chunks(ql);
    const size_t need = align_up(size_t(nch + 1) * 4) + size_t(nch + 1) * 8 + 16;
    ensure(&c->qtmp, &c->qtmp_bytes, need, c, "cudaMalloc(quant tmp)");
    char* b = static_cast<char*>(c->qtmp);
    uint32_t* counts = reinterpret_cast<uint32_t*>(b);
    uint64_t* offsets = reinterpret_cast<uint64_t*>(b + align_up(size_t(nch + 1) * 4));
    int* flags = reinterpret_cast<int*>(offsets + nch + 1);
    cuda_check(cudaMemsetAsync(flags, 0, sizeof(int), c->stream), "memset");
    cudaError_t e;
    if (dtype == MGRX_F32)
      e = quantize_pass1<float>(static_cast<const float*>(d_coeffs), d_labels, counts, offsets, flags, ql, exec(c));
    else
      e = quantize_pass1<double>(static_cast<const double*>(d_coeffs), d_labels, counts, offsets, flags, ql,
                                 exec(c));
    cuda_check(e, "quantize");
    // the ordered outlier pass runs without waiting for the total: it
    // writes the outliers that fit the capacity; one readback then gives the
    // count (capacity exceeded: the caller retries with the exact count)
    if (d_opos && d_oval && capacity > 0) {
      if (dtype == MGRX_F32)
        e = quantize_pass2<float>(static_cast<const float*>(d_coeffs), counts, offsets, d_opos,
                                  static_cast<float*>(d_oval), capacity, ql, exec(c));
      else
        e = quantize_pass2<double>(static_cast<const double*>(d_coeffs), counts, offsets, d_opos,
                                   static_cast<double*>(d_oval), capacity, ql, exec(c));
      cuda_check(e, "quantize outliers");
    }
    uint64_t* hp = static_cast<uint64_t*>(c->pinned);
    cuda_check(cudaMemcpyAsync(hp, offsets + nch, 8, cudaMemcpyDeviceToHost, c->stream), "readback");
    cuda_check(cudaMemcpyAsync(hp + 1, flags, 4, cudaMemcpyDeviceToHost, c->stream), "readback");
    cuda_check(cudaStreamSynchronize(c->stream), "quantize sync");
    const uint64_t total = hp[0];
    const int flag = *reinterpret_cast<int*>(hp + 1);
    *n_outliers = total;
    if (flag) fail(MGRX_NONFINITE_DATA, "non-finite value in quantizer input");
    if (total > capacity) fail(MGRX_CAPACITY_EXCEEDED, "%llu outliers exceed capacity %llu",
                               (unsigned long long)total, (unsigned long long)capacity);
    if (total > 0 && (!d_opos || !d_oval)) fail(MGRX_INVALID_ARGUMENT, "null outlier buffers");
  });
}

int mgrx_gpu_dequantize(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int stop,
                        const double* q, const int32_t* d_labels, const uint64_t* d_opos, const void* d_oval,
                        uint64_t n_outliers, void* d_coeffs) {
  return guarded(c, [&] {
    if (!dims || !q || !d_labels || !d_coeffs) fail(MGRX_INVALID_ARGUMENT, "null argument");
    if (n_outliers && (!d_opos || !d_oval)) fail(MGRX_INVALID_ARGUMENT, "null outlier buffers");
    Plan* p = get_plan(c, dtype, nd, dims, levels, stop);
    QuantLevels ql = quant_levels(*p, q);
    cudaError_t e;
    if (dtype == MGRX_F32)
      e = dequantize_run<float>(d_labels, d_opos, static_cast<const float*>(d_oval), n_outliers,
                                static_cast<float*>(d_coeffs), ql, exec(c));
    else
      e = dequantize_run<double>(d_labels, d_opos, static_cast<const double*>(d_oval), n_outliers,
                                 static_cast<double*>(d_coeffs), ql, exec(c));
    cuda_check(e, "dequantize");
  });
}

}  // extern "C"

// Quantizer scratch of a call: per-chunk outlier counts, their scan, flags.
struct QuantTmp {
  uint32_t* counts;
  uint64_t* offsets;
  int* flags;
  int64_t nch;
};
static QuantTmp quant_tmp(mgrx_gpu_ctx* c, const QuantLevels& ql) {
  const int64_t nch = quant_num_chunks(ql);
  const size_t need = align_up(size_t(nch + 1) * 4) + size_t(nch + 1) * 8 + 16;
  ensure(&c->qtmp, &c->qtmp_bytes, need, c, "cudaMalloc(quant tmp)");
  char* b = static_cast<char*>(c->qtmp);
  QuantTmp t;
  t.counts = reinterpret_cast<uint32_t*>(b);
  t.offsets = reinterpret_cast<uint64_t*>(b + align_up(size_t(nch + 1) * 4));
  t.flags = reinterpret_cast<int*>(t.offsets + nch + 1);
  t.nch = nch;
  return t;
}

// Runs the body with the context's stream switched to `s` (the level drivers
// launch on c->stream).
struct StreamSwap {
  mgrx_gpu_ctx* c;
  cudaStream_t saved;
  StreamSwap(mgrx_gpu_ctx* c_, cudaStream_t s) : c(c_), saved(c_->stream) { c->stream = s; }
  ~StreamSwap() { c->stream = saved; }
};

template <typename T>
static void decompose_quantize_impl(mgrx_gpu_ctx* c, Plan& p, const T* d_field, const double* q, T* d_coeffs,
                                    int32_t* d_labels, uint64_t* d_opos, T* d_oval, uint64_t capacity,
                                    uint64_t* n_outliers) {
  const Hierarchy& h = p.h;
  const int L = h.L;
  QuantLevels ql = quant_levels(p, q);
  QuantTmp qt = quant_tmp(c, ql);
  cuda_check(cudaMemsetAsync(qt.flags, 0, sizeof(int), c->stream), "memset");
  // chunks [split, nch) lie inside the finest shell: they are quantized on a
  // low-priority side stream as soon as the finest level's plane pass has
  // written that shell, under the rest of the decomposition (the finest
  // level's solves and every coarser level: latency-bound, little HBM
  // traffic), which runs on the high-priority chain stream
  const bool overlap = L > p.stop && c->path == 0 && p.fused[L].enabled && !c->profiling;
  int64_t split = qt.nch;
  if (overlap) {
    ensure_side(c, L + 1);
    split = std::min(qt.nch, quant_chunk_of(ql, h.node[L - 1]));
    cuda_check(cudaEventRecord(c->fork, c->stream), "cudaEventRecord(fork)");
    cuda_check(cudaStreamWaitEvent(c->chain, c->fork, 0), "cudaStreamWaitEvent");
    bool used = false;
    {
      StreamSwap sw(c, c->chain);
      decompose_impl<T>(c, p, d_field, d_coeffs, nullptr, c->lvl_done[L], &used);
    }
    cuda_check(cudaEventRecord(c->join, c->chain), "cudaEventRecord(join)");
    if (used) {
      cudaStream_t sd = c->side[0];
      cuda_check(cudaStreamWaitEvent(sd, c->lvl_done[L], 0), "cudaStreamWaitEvent");
      cuda_check(quantize_labels_range<T>(d_coeffs, d_labels, qt.counts, qt.flags, ql, split, qt.nch,
                                          exec_on(c, sd, L)),
                 "quantize finest shell");
      cuda_check(cudaEventRecord(c->lvl_done[0], sd), "cudaEventRecord");
      cuda_check(cudaStreamWaitEvent(c->stream, c->lvl_done[0], 0), "cudaStreamWaitEvent");
    } else {
      split = qt.nch;
    }
    cuda_check(cudaStreamWaitEvent(c->stream, c->join, 0), "cudaStreamWaitEvent");
  } else {
    decompose_impl<T>(c, p, d_field, d_coeffs, nullptr);
  }
  cuda_check(quantize_labels_range<T>(d_coeffs, d_labels, qt.counts, qt.flags, ql, 0, split, exec(c)),
             "quantize");
  cuda_check(quantize_scan(qt.counts, qt.offsets, ql, exec(c)), "quantize scan");
  if (d_opos && d_oval && capacity > 0)
    cuda_check(quantize_pass2<T>(d_coeffs, qt.counts, qt.offsets, d_opos, d_oval, capacity, ql, exec(c)),
               "quantize outliers");
  uint64_t* hp = static_cast<uint64_t*>(c->pinned);
  cuda_check(cudaMemcpyAsync(hp, qt.offsets + qt.nch, 8, cudaMemcpyDeviceToHost, c->stream), "readback");
  cuda_check(cudaMemcpyAsync(hp + 1, qt.flags, 4, cudaMemcpyDeviceToHost, c->stream), "readback");
  cuda_check(cudaStreamSynchronize(c->stream), "quantize sync");
  const uint64_t total = hp[0];
  const int flag = *reinterpret_cast<int*>(hp + 1);
  *n_outliers = total;
  if (flag) fail(MGRX_NONFINITE_DATA, "non-finite value in quantizer input");
  if (total > capacity)
    fail(MGRX_CAPACITY_EXCEEDED, "%llu outliers exceed capacity %llu", (unsigned long long)total,
         (unsigned long long)capacity);
  if (total > 0 && (!d_opos || !d_oval)) fail(MGRX_INVALID_ARGUMENT, "null outlier buffers");
}

template <typename T>
static void dequantize_recompose_impl(mgrx_gpu_ctx* c, Plan& p, const double* q, const int32_t* d_labels,
                                      const uint64_t* d_opos, const T* d_oval, uint64_t n_outliers, T* d_coeffs,
                                      T* d_field) {
  const Hierarchy& h = p.h;
  const int L = h.L;
  QuantLevels ql = quant_levels(p, q);
  const int64_t nch = quant_num_chunks(ql);
  // the finest shell's labels are dequantized (and its outliers restored) on
  // the stream of the finest level's correction, which reads only that
  // shell, after the coarser shells, whose levels' work then runs beside it
  const bool overlap = L > p.stop && c->path == 0 && p.fused[L].enabled && !c->profiling;
  if (!overlap) {
    cuda_check(dequantize_run<T>(d_labels, d_opos, d_oval, n_outliers, d_coeffs, ql, exec(c)), "dequantize");
    recompose_impl<T>(c, p, d_coeffs, d_field, nullptr);
    return;
  }
  const int64_t split = std::min(nch, quant_chunk_of(ql, h.node[L - 1]));
  cuda_check(dequantize_range<T>(d_labels, d_opos, d_oval, n_outliers, d_coeffs, ql, 0, split, exec(c)),
             "dequantize");
  c->rec_pre_finest = [&](cudaStream_t sd) {
    cuda_check(dequantize_range<T>(d_labels, d_opos, d_oval, n_outliers, d_coeffs, ql, split, nch,
                                   exec_on(c, sd, L)),
               "dequantize finest shell");
  };
  try {
    recompose_impl<T>(c, p, d_coeffs, d_field, nullptr);
  } catch (...) {
    c->rec_pre_finest = nullptr;
    throw;
  }
  c->rec_pre_finest = nullptr;
}

extern "C" {

int mgrx_gpu_decompose_quantize(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int stop,
                                const void* d_field, const double* q, void* d_coeffs, int32_t* d_labels,
                                uint64_t* d_opos, void* d_oval, uint64_t capacity, uint64_t* n_outliers) {
  return guarded(c, [&] {
    if (!dims || !q || !d_field || !d_coeffs || !d_labels || !n_outliers)
      fail(MGRX_INVALID_ARGUMENT, "null argument");
    Plan* p = get_plan(c, dtype, nd, dims, levels, stop);
    for (int l = 0; l <= p->h.L; ++l)
      if (!(q[l] > 0.0) || !std::isfinite(q[l])) fail(MGRX_INVALID_BUDGET, "bad bin width at level %d", l);
    if (dtype == MGRX_F32)
      decompose_quantize_impl<float>(c, *p, static_cast<const float*>(d_field), q, static_cast<float*>(d_coeffs),
                                     d_labels, d_opos, static_cast<float*>(d_oval), capacity, n_outliers);
    else
      decompose_quantize_impl<double>(c, *p, static_cast<const double*>(d_field), q,
                                      static_cast<double*>(d_coeffs), d_labels, d_opos,
                                      static_cast<double*>(d_oval), capacity, n_outliers);
  });
}

int mgrx_gpu_dequantize_recompose(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int stop,
                                  const double* q, const int32_t* d_labels, const uint64_t* d_opos,
                                  const void* d_oval, uint64_t n_outliers, void* d_coeffs, void* d_field) {
  return guarded(c, [&] {
    if (!dims || !q || !d_labels || !d_coeffs || !d_field) fail(MGRX_INVALID_ARGUMENT, "null argument");
    if (n_outliers && (!d_opos || !d_oval)) fail(MGRX_INVALID_ARGUMENT, "null outlier buffers");
    Plan* p = get_plan(c, dtype, nd, dims, levels, stop);
    if (dtype == MGRX_F32)
      dequantize_recompose_impl<float>(c, *p, q, d_labels, d_opos, static_cast<const float*>(d_oval), n_outliers,
                                       static_cast<float*>(d_coeffs), static_cast<float*>(d_field));
    else
      dequantize_recompose_impl<double>(c, *p, q, d_labels, d_opos, static_cast<const double*>(d_oval),
                                        n_outliers, static_cast<double*>(d_coeffs), static_cast<double*>(d_field));
  });
}

}  // extern "C"

extern "C" {

static int host_roundtrip(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int stop,
                          const void* h_in, void* h_out, bool dec) {
  return guarded(c, [&] {
    if (!dims || !h_in || !h_out) fail(MGRX_INVALID_ARGUMENT, "null argument");
    Plan* p = get_plan(c, dtype, nd, dims, levels, stop);
    const size_t bytes = size_t(p->h.node[p->h.L]) * p->esize;
    ensure(&c->io, &c->io_bytes, 2 * align_up(bytes), c, "cudaMalloc(io)");
    char* din = static_cast<char*>(c->io);
    char* dout = din + align_up(bytes);
    cuda_check(cudaMemcpyAsync(din, h_in, bytes, cudaMemcpyHostToDevice, c->stream), "H2D");
    if (dtype == MGRX_F32) {
      if (dec) decompose_impl<float>(c, *p, reinterpret_cast<float*>(din), reinterpret_cast<float*>(dout), nullptr);
      else recompose_impl<float>(c, *p, reinterpret_cast<float*>(din), reinterpret_cast<float*>(dout), nullptr);
    } else {
      if (dec) decompose_impl<double>(c, *p, reinterpret_cast<double*>(din), reinterpret_cast<double*>(dout), nullptr);
      else recompose_impl<double>(c, *p, reinterpret_cast<double*>(din), reinterpret_cast<double*>(dout), nullptr);
    }
    cuda_check(cudaMemcpyAsync(h_out, dout, bytes, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
  });
}

int mgrx_host_quantize(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int stop,
                       const double* q, const void* h_coeffs, int32_t* h_labels, uint64_t* h_opos, void* h_oval,
                       uint64_t capacity, uint64_t* n_outliers) {
  int rc = guarded(c, [&] {
    if (!dims || !q || !h_coeffs || !h_labels || !n_outliers) fail(MGRX_INVALID_ARGUMENT, "null argument");
    Plan* p = get_plan(c, dtype, nd, dims, levels, stop);
    const size_t n = size_t(p->h.node[p->h.L]);
    const size_t base = stop == 0 ? 0 : size_t(p->h.node[stop]);
    const size_t es = p->esize;
    const size_t need = align_up(n * es) + align_up((n - base) * 4) + align_up(n * 8) + align_up(n * es);
    ensure(&c->io, &c->io_bytes, need, c, "cudaMalloc(io)");
    char* b = static_cast<char*>(c->io);
    char* dc = b;
    int32_t* dl = reinterpret_cast<int32_t*>(b + align_up(n * es));
    uint64_t* dp = reinterpret_cast<uint64_t*>(b + align_up(n * es) + align_up((n - base) * 4));
    char* dv = reinterpret_cast<char*>(dp) + align_up(n * 8);
    cuda_check(cudaMemcpyAsync(dc, h_coeffs, n * es, cudaMemcpyHostToDevice, c->stream), "H2D");
    const int r = mgrx_gpu_quantize(c, dtype, nd, dims, levels, stop, q, dc, dl, dp, dv, n, n_outliers);
    if (r != MGRX_OK) throw Fail{r, c->last_error};
    if (*n_outliers > capacity) fail(MGRX_CAPACITY_EXCEEDED, "%llu outliers exceed capacity %llu",
                                     (unsigned long long)*n_outliers, (unsigned long long)capacity);
    cuda_check(cudaMemcpyAsync(h_labels, dl, (n - base) * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    if (*n_outliers) {
      cuda_check(cudaMemcpyAsync(h_opos, dp, *n_outliers * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
      cuda_check(cudaMemcpyAsync(h_oval, dv, *n_outliers * es, cudaMemcpyDeviceToHost, c->stream), "D2H");
    }
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
  });
  return rc;
}

int mgrx_host_dequantize(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int stop,
                         const double* q, const int32_t* h_labels, const uint64_t* h_opos, const void* h_oval,
                         uint64_t n_outliers, void* h_coeffs) {
  return guarded(c, [&] {
    if (!dims || !q || !h_labels || !h_coeffs) fail(MGRX_INVALID_ARGUMENT, "null argument");
    if (n_outliers && (!h_opos || !h_oval)) fail(MGRX_INVALID_ARGUMENT, "null outlier buffers");
    Plan* p = get_plan(c, dtype, nd, dims, levels, stop);
    const size_t n = size_t(p->h.node[p->h.L]);
    const size_t base = stop == 0 ? 0 : size_t(p->h.node[stop]);
    const size_t es = p->esize;
    const size_t no = size_t(n_outliers);
    const size_t need = align_up(n * es) + align_up((n - base) * 4) + align_up(no * 8 + 8) + align_up(no * es + 8);
    ensure(&c->io, &c->io_bytes, need, c, "cudaMalloc(io)");
    char* b = static_cast<char*>(c->io);
    char* dc = b;
    int32_t* dl = reinterpret_cast<int32_t*>(b + align_up(n * es));
    uint64_t* dp = reinterpret_cast<uint64_t*>(b + align_up(n * es) + align_up((n - base) * 4));
    char* dv = reinterpret_cast<char*>(dp) + align_up(no * 8 + 8);
    // the coarse block of a tail dequantize is preserved: start from the caller's buffer
    cuda_check(cudaMemcpyAsync(dc, h_coeffs, n * es, cudaMemcpyHostToDevice, c->stream), "H2D");
    cuda_check(cudaMemcpyAsync(dl, h_labels, (n - base) * 4, cudaMemcpyHostToDevice, c->stream), "H2D");
    if (no) {
      cuda_check(cudaMemcpyAsync(dp, h_opos, no * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
      cuda_check(cudaMemcpyAsync(dv, h_oval, no * es, cudaMemcpyHostToDevice, c->stream), "H2D");
    }
    const int r = mgrx_gpu_dequantize(c, dtype, nd, dims, levels, stop, q, dl, dp, dv, n_outliers, dc);
    if (r != MGRX_OK) throw Fail{r, c->last_error};
    cuda_check(cudaMemcpyAsync(h_coeffs, dc, n * es, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
  });
}

// decompress_field's ★ pair from host buffers (pipeline.hpp:235-260): the
// labels, the outliers and (stop > 0) the decoded coarse block go to the GPU,
// dequantize + recompose run there back to back, only the field comes back
// (the two host calls would move the N coefficients down and up again).
int mgrx_host_decompress(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int stop,
                         const double* q, const int32_t* h_labels, const uint64_t* h_opos, const void* h_oval,
                         uint64_t n_outliers, const void* h_coarse, void* h_field) {
  return guarded(c, [&] {
    if (!dims || !q || !h_labels || !h_field) fail(MGRX_INVALID_ARGUMENT, "null argument");
    if (n_outliers && (!h_opos || !h_oval)) fail(MGRX_INVALID_ARGUMENT, "null outlier buffers");
    Plan* p = get_plan(c, dtype, nd, dims, levels, stop);
    if (stop > 0 && !h_coarse) fail(MGRX_INVALID_ARGUMENT, "a tail stream needs the coarse block");
    const size_t n = size_t(p->h.node[p->h.L]);
    const size_t base = stop == 0 ? 0 : size_t(p->h.node[stop]);
    const size_t es = p->esize;
    const size_t no = size_t(n_outliers);
    const size_t need =
        2 * align_up(n * es) + align_up((n - base) * 4) + align_up(no * 8 + 8) + align_up(no * es + 8);
    ensure(&c->io, &c->io_bytes, need, c, "cudaMalloc(io)");
    char* b = static_cast<char*>(c->io);
    char* dc = b;
    char* df = b + align_up(n * es);
    int32_t* dl = reinterpret_cast<int32_t*>(df + align_up(n * es));
    uint64_t* dp = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(dl) + align_up((n - base) * 4));
    char* dv = reinterpret_cast<char*>(dp) + align_up(no * 8 + 8);
    if (base) cuda_check(cudaMemcpyAsync(dc, h_coarse, base * es, cudaMemcpyHostToDevice, c->stream), "H2D");
    cuda_check(cudaMemcpyAsync(dl, h_labels, (n - base) * 4, cudaMemcpyHostToDevice, c->stream), "H2D");
    if (no) {
      cuda_check(cudaMemcpyAsync(dp, h_opos, no * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
      cuda_check(cudaMemcpyAsync(dv, h_oval, no * es, cudaMemcpyHostToDevice, c->stream), "H2D");
    }
    const int r = mgrx_gpu_dequantize_recompose(c, dtype, nd, dims, levels, stop, q, dl, dp, dv, n_outliers, dc, df);
    if (r != MGRX_OK) throw Fail{r, c->last_error};
    cuda_check(cudaMemcpyAsync(h_field, df, n * es, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
  });
}

int mgrx_host_decompose(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int stop,
                        const void* h_field, void* h_out) {
  return host_roundtrip(c, dtype, nd, dims, levels, stop, h_field, h_out, true);
}

int mgrx_host_recompose(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int stop,
                        const void* h_coeffs, void* h_field) {
  return host_roundtrip(c, dtype, nd, dims, levels, stop, h_coeffs, h_field, false);
}

}  // extern "C"

namespace {
// decompose_with (transform.hpp:485-506) with the reference's adaptive
// decider (choose_stop, adaptive.hpp:99-104) evaluated on the GPU: the level
// blocks never leave the device.  Each level step decomposes the level block
// as a field of l levels stopped at l - 1 (the same arithmetic as the full
// decompose, and as the host decompose_with of include/mgrx_b200.hpp).
// Device version: d_field (read only) -> d_out (level-centric), *stop_out.
template <typename T>
void decompose_adaptive_dev(mgrx_gpu_ctx* c, int nd, const uint64_t* dims, int levels, const T* d_field,
                            const double* e_lvl, const double* pen_lvl, const double* lz_lvl, int step, int min_stop,
                            T* out, int* stop_out) {
  const Hierarchy h = make_hierarchy(nd, dims, levels);
  const int L = h.L;
  if (min_stop < 0 || min_stop > L) fail(MGRX_INVALID_LEVEL, "stop level out of range");
  const int code = sizeof(T) == 4 ? MGRX_F32 : MGRX_F64;
  const size_t N = size_t(h.node[L]);
  T *blk = nullptr, *nxt = nullptr;
  cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&blk), N * sizeof(T), c->stream), "cudaMalloc");
  cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&nxt), N * sizeof(T), c->stream), "cudaMalloc");
  struct Free {
    mgrx_gpu_ctx* c;
    void* p[2];
    ~Free() {
      for (void* q : p)
        if (q) cudaFreeAsync(q, c->stream);
    }
  } fr{c, {blk, nxt}};
  cuda_check(cudaMemcpyAsync(blk, d_field, N * sizeof(T), cudaMemcpyDeviceToDevice, c->stream), "copy field");
  int stop = min_stop;
  for (int l = L; l > min_stop; --l) {
    uint64_t dl[kMaxD];
    for (int i = 0; i < nd; ++i) dl[i] = uint64_t(h.dims[l][i]);
    int st = 0;
    const int rc = mgrx_gpu_choose_stop(c, code, nd, dl, blk, e_lvl[l], pen_lvl + size_t(l) * nd, lz_lvl[l], step,
                                        nullptr, &st);
    if (rc != MGRX_OK) fail(rc, "%s", c->last_error.c_str());
    if (st) {
      stop = l;
      break;
    }
    Plan* p = get_plan(c, code, nd, dl, l, l - 1);
    decompose_impl<T>(c, *p, blk, nxt, nullptr);  // nxt = [coarse block of l - 1 | shell of level l]
    const size_t nc = size_t(h.node[l - 1]), nl = size_t(h.node[l]);
    cuda_check(cudaMemcpyAsync(out + nc, nxt + nc, (nl - nc) * sizeof(T), cudaMemcpyDeviceToDevice, c->stream),
               "copy shell");
    std::swap(blk, nxt);
  }
  cuda_check(cudaMemcpyAsync(out, blk, size_t(h.node[stop]) * sizeof(T), cudaMemcpyDeviceToDevice, c->stream),
             "copy coarse");
  *stop_out = stop;
}

template <typename T>
void decompose_adaptive_impl(mgrx_gpu_ctx* c, int nd, const uint64_t* dims, int levels, const T* h_field,
                             const double* e_lvl, const double* pen_lvl, const double* lz_lvl, int step,
                             int min_stop, T* h_out, int* stop_out) {
  const Hierarchy h = make_hierarchy(nd, dims, levels);
  const size_t N = size_t(h.node[h.L]);
  T *din = nullptr, *dout = nullptr;
  cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&din), N * sizeof(T), c->stream), "cudaMalloc");
  cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&dout), N * sizeof(T), c->stream), "cudaMalloc");
  struct Free {
    mgrx_gpu_ctx* c;
    void* p[2];
    ~Free() {
      for (void* q : p)
        if (q) cudaFreeAsync(q, c->stream);
    }
  } fr{c, {din, dout}};
  cuda_check(cudaMemcpyAsync(din, h_field, N * sizeof(T), cudaMemcpyHostToDevice, c->stream), "H2D");
  decompose_adaptive_dev<T>(c, nd, dims, levels, din, e_lvl, pen_lvl, lz_lvl, step, min_stop, dout, stop_out);
  cuda_check(cudaMemcpyAsync(h_out, dout, N * sizeof(T), cudaMemcpyDeviceToHost, c->stream), "D2H");
  cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
}

// Range and finiteness of n device values (check_finite, pipeline.hpp:113-118).
template <typename T>
void field_stats_run(mgrx_gpu_ctx* c, const T* d, int64_t n, double* lo, double* hi, uint64_t* first_bad) {
  *lo = INFINITY;
  *hi = -INFINITY;
  *first_bad = uint64_t(n);
  if (n <= 0) return;
  const int nb = field_stats_blocks(n);
  void* p = nullptr;
  cuda_check(cudaMallocAsync(&p, size_t(nb) * 24, c->stream), "cudaMallocAsync");
  double* bmin = static_cast<double*>(p);
  double* bmax = bmin + nb;
  auto* bbad = reinterpret_cast<unsigned long long*>(bmax + nb);
  cudaError_t e = field_stats<T>(d, n, bmin, bmax, bbad, exec(c));
  std::vector<double> h(size_t(nb) * 3);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), p, size_t(nb) * 24, cudaMemcpyDeviceToHost, c->stream);
  cudaFreeAsync(p, c->stream);
  cuda_check(e, "field stats");
  cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  for (int b = 0; b < nb; ++b) {
    *lo = std::min(*lo, h[size_t(b)]);
    *hi = std::max(*hi, h[size_t(nb + b)]);
    uint64_t bad;
    std::memcpy(&bad, &h[size_t(2 * nb + b)], 8);
    *first_bad = std::min<uint64_t>(*first_bad, bad);
  }
}

// check_finite / range fused into the finest level's first plane pass:
// nf_flag = {u32 non-finite flag, pad, u64 min, u64 max} (order-preserving
// images of the fp64 values, see fused3d.cu ordered_bits).
uint64_t ordered_bits_host(double x) {
  uint64_t b;
  std::memcpy(&b, &x, 8);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
double from_ordered_bits(uint64_t o) {
  const uint64_t b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
  double x;
  std::memcpy(&x, &b, 8);
  return x;
}
void nf_arm(mgrx_gpu_ctx* c) {
  if (!c->nf_flag) cuda_check(cudaMalloc(reinterpret_cast<void**>(&c->nf_flag), 64), "cudaMalloc(flag)");
  static const uint64_t init[3] = {0, ordered_bits_host(INFINITY), ordered_bits_host(-INFINITY)};
  cuda_check(cudaMemcpyAsync(c->nf_flag, init, sizeof init, cudaMemcpyHostToDevice, c->stream), "init flag");
  c->nf_used = false;
  c->nf_armed = true;
}
// after the decompose: the fused stats when the finest level carried them
// (true), else false (the caller runs field_stats)
bool nf_read(mgrx_gpu_ctx* c, unsigned* flag, double* lo, double* hi) {
  c->nf_armed = false;
  if (!c->nf_used) return false;
  uint64_t h[3];
  cuda_check(cudaMemcpyAsync(h, c->nf_flag, sizeof h, cudaMemcpyDeviceToHost, c->stream), "D2H");
  cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  *flag = unsigned(h[0] & 0xffffffffu);
  *lo = from_ordered_bits(h[1]);
  *hi = from_ordered_bits(h[2]);
  return true;
}

// compress's device part (pipeline.hpp:130-196 up to the sections): the
// field goes to the GPU once; decompose (fixed or adaptive stop),
// quantize and every level's encode_labels run there; the encoded label
// sections, the outliers and (stop > 0) the coarse block come back.
template <typename T>
void compress_core(mgrx_gpu_ctx* c, int nd, const uint64_t* dims, int levels, const T* h_field, const double* q,
                   int adaptive, int force_stop, const double* e_lvl, const double* pen_lvl, const double* lz_lvl,
                   uint8_t* h_sec, uint64_t sec_cap, uint64_t* sec_sizes, uint64_t* h_opos, T* h_oval,
                   uint64_t o_cap, uint64_t* n_out, T* h_coarse, int* stop_out) {
  const Hierarchy h = make_hierarchy(nd, dims, levels);
  const int L = h.L;
  const int code = sizeof(T) == 4 ? MGRX_F32 : MGRX_F64;
  const size_t N = size_t(h.node[L]);
  std::vector<void*> bufs;
  struct Free {
    mgrx_gpu_ctx* c;
    std::vector<void*>* b;
    ~Free() {
      for (void* q : *b) cudaFreeAsync(q, c->stream);
    }
  } fr{c, &bufs};
  auto dalloc = [&](size_t bytes) {
    void* p = nullptr;
    cuda_check(cudaMallocAsync(&p, std::max<size_t>(bytes, 16), c->stream), "cudaMallocAsync");
    bufs.push_back(p);
    return p;
  };
  T* dfield = static_cast<T*>(dalloc(N * sizeof(T)));
  T* dco = static_cast<T*>(dalloc(N * sizeof(T)));
  cuda_check(cudaMemcpyAsync(dfield, h_field, N * sizeof(T), cudaMemcpyHostToDevice, c->stream), "H2D");
  // check_finite (pipeline.hpp:132): fused into the finest level's first
  // pass when that level runs on the fused 3-D path (no extra read of the
  // field); otherwise a separate pass over the device copy.  On a non-finite
  // value the reference's error (first offset) is raised either way.
  auto check_finite_pass = [&]() {
    double lo, hi;
    uint64_t bad;
    field_stats_run<T>(c, dfield, int64_t(N), &lo, &hi, &bad);
    if (bad < N) fail(MGRX_NONFINITE_DATA, "non-finite value at offset %llu", (unsigned long long)bad);
  };
  nf_arm(c);
  c->nf_armed = force_stop < 0 || force_stop < L;
  struct Disarm {
    mgrx_gpu_ctx* c;
    ~Disarm() { c->nf_armed = false; }
  } disarm{c};
  int stop = 0;
  if (force_stop >= 0) {
    if (force_stop > L) fail(MGRX_INVALID_LEVEL, "forced stop level out of range");
    stop = force_stop;
  } else if (adaptive) {
    decompose_adaptive_dev<T>(c, nd, dims, L, dfield, e_lvl, pen_lvl, lz_lvl, 8, 0, dco, &stop);
  }
  *stop_out = stop;
  for (int l = 0; l <= L; ++l) sec_sizes[l] = 0;
  *n_out = 0;
  if (stop == L) {  // Lorenzo only (the caller codes the field)
    check_finite_pass();
    return;
  }
  if (!(force_stop < 0 && adaptive)) {
    const int rc = mgrx_gpu_decompose(c, code, nd, dims, L, stop, dfield, dco);
    if (rc != MGRX_OK) fail(rc, "%s", c->last_error.c_str());
  }
  {
    unsigned flag = 0;
    double lo, hi;
    if (nf_read(c, &flag, &lo, &hi)) {
      if (flag) check_finite_pass();  // locates the first offset and raises
    } else {
      check_finite_pass();
    }
  }
  const size_t base = stop == 0 ? 0 : size_t(h.node[stop]);
  int32_t* dlab = static_cast<int32_t*>(dalloc((N - base) * 4));
  uint64_t cap = 1 << 16, nout = 0;
  uint64_t* dpos = nullptr;
  T* dval = nullptr;
  for (;;) {
    dpos = static_cast<uint64_t*>(dalloc(cap * 8));
    dval = static_cast<T*>(dalloc(cap * sizeof(T)));
    const int rc = mgrx_gpu_quantize(c, code, nd, dims, L, stop, q, dco, dlab, dpos, dval, cap, &nout);
    if (rc == MGRX_CAPACITY_EXCEEDED) {
      cap = nout;
      continue;
    }
    if (rc != MGRX_OK) fail(rc, "%s", c->last_error.c_str());
    break;
  }
  *n_out = nout;
  if (nout > o_cap) fail(MGRX_CAPACITY_EXCEEDED, "%llu outliers exceed capacity %llu", (unsigned long long)nout,
                         (unsigned long long)o_cap);
  if (nout) {
    cuda_check(cudaMemcpyAsync(h_opos, dpos, nout * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaMemcpyAsync(h_oval, dval, nout * sizeof(T), cudaMemcpyDeviceToHost, c->stream), "D2H");
  }
  // per level: encode_labels of the level's labels (0 = coarsest)
  uint64_t at = 0, used = 0;
  for (int l = stop == 0 ? 0 : stop + 1; l <= L; ++l) {
    const uint64_t cnt = uint64_t(h.delta[l]);
    uint64_t sz = 0;
    const int rc = mgrx_gpu_encode_labels(c, dlab + at, cnt, h_sec + used, sec_cap - used, &sz);
    if (rc == MGRX_CAPACITY_EXCEEDED) fail(rc, "section capacity exceeded");
    if (rc != MGRX_OK) fail(rc, "%s", c->last_error.c_str());
    sec_sizes[l] = sz;
    used += sz;
    at += cnt;
  }
  if (stop > 0 && h_coarse)
    cuda_check(cudaMemcpyAsync(h_coarse, dco, size_t(h.node[stop]) * sizeof(T), cudaMemcpyDeviceToHost, c->stream),
               "D2H");
  cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
}
}  // namespace

extern "C" {

int mgrx_host_lorenzo(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, const void* h_block, double e,
                      uint8_t* h_enc, uint64_t enc_capacity, uint64_t* enc_size, uint64_t* h_outlier_pos,
                      void* h_outlier_val, uint64_t outlier_capacity, uint64_t* n_outliers) {
  return guarded(c, [&] {
    if (!dims || !h_block || !enc_size || !n_outliers) fail(MGRX_INVALID_ARGUMENT, "null argument");
    if (nd < 1 || nd > kMaxD) fail(MGRX_INVALID_DIMS, "lorenzo: rank out of range");
    if (!(e > 0.0) || !std::isfinite(e)) fail(MGRX_INVALID_BUDGET, "error bound must be positive");
    const size_t es = dtype == MGRX_F32 ? 4 : 8;
    int64_t n[kMaxD], N = 1, H = 1;
    for (int i = 0; i < nd; ++i) {
      n[i] = int64_t(dims[i]);
      if (n[i] < 1) fail(MGRX_INVALID_DIMS, "lorenzo: empty extent");
      N *= n[i];
      H += n[i] - 1;
    }
    if (N > int64_t(0xffffffffu)) fail(MGRX_INVALID_DIMS, "lorenzo: block too large");
    // positions grouped by hyperplane sum(index) (counting sort, position order within)
    std::vector<uint32_t> hs(size_t(H) + 1, 0), order(static_cast<size_t>(N));
    {
      std::vector<uint32_t> hof(static_cast<size_t>(N));
      int64_t idx[kMaxD] = {0};
      int64_t h = 0;
      for (int64_t p = 0; p < N; ++p) {
        hof[size_t(p)] = uint32_t(h);
        ++hs[size_t(h) + 1];
        for (int i = nd - 1; i >= 0; --i) {  // odometer, h tracks sum(index)
          if (++idx[i] < n[i]) {
            ++h;
            break;
          }
          h -= idx[i] - 1;
          idx[i] = 0;
        }
      }
      for (int64_t k = 0; k < H; ++k) hs[size_t(k) + 1] += hs[size_t(k)];
      std::vector<uint32_t> next(hs.begin(), hs.end() - 1);
      for (int64_t p = 0; p < N; ++p) order[next[hof[size_t(p)]]++] = uint32_t(p);
    }
    std::vector<void*> bufs;
    struct Free {
      mgrx_gpu_ctx* c;
      std::vector<void*>* b;
      ~Free() {
        for (void* q : *b) cudaFreeAsync(q, c->stream);
      }
    } fr{c, &bufs};
    auto dalloc = [&](size_t bytes) {
      void* q = nullptr;
      cuda_check(cudaMallocAsync(&q, std::max<size_t>(bytes, 16), c->stream), "cudaMallocAsync");
      bufs.push_back(q);
      return q;
    };
    void* dx = dalloc(size_t(N) * es);
    void* drec = dalloc(size_t(N) * es);
    auto* dord = static_cast<uint32_t*>(dalloc(size_t(N) * 4));
    auto* dhs = static_cast<uint32_t*>(dalloc((size_t(H) + 1) * 4));
    auto* dlab = static_cast<int32_t*>(dalloc(size_t(N) * 4));
    auto* dfl = static_cast<uint8_t*>(dalloc(size_t(N)));
    const uint64_t cap = std::max<uint64_t>(outlier_capacity, 1);
    auto* dpos = static_cast<uint64_t*>(dalloc(cap * 8));
    void* dval = dalloc(cap * es);
    auto* dcnt = static_cast<unsigned long long*>(dalloc(8));
    cuda_check(cudaMemcpyAsync(dx, h_block, size_t(N) * es, cudaMemcpyHostToDevice, c->stream), "H2D");
    cuda_check(cudaMemcpyAsync(dord, order.data(), size_t(N) * 4, cudaMemcpyHostToDevice, c->stream), "H2D");
    cuda_check(cudaMemcpyAsync(dhs, hs.data(), (size_t(H) + 1) * 4, cudaMemcpyHostToDevice, c->stream), "H2D");
    cudaError_t err;
    if (dtype == MGRX_F32)
      err = lorenzo_run<float>(static_cast<const float*>(dx), nd, n, dord, dhs, int(H), e, dlab, dfl,
                               static_cast<float*>(drec), dpos, static_cast<float*>(dval), cap, dcnt, exec(c));
    else
      err = lorenzo_run<double>(static_cast<const double*>(dx), nd, n, dord, dhs, int(H), e, dlab, dfl,
                                static_cast<double*>(drec), dpos, static_cast<double*>(dval), cap, dcnt, exec(c));
    cuda_check(err, "lorenzo");
    unsigned long long cnt = 0;
    cuda_check(cudaMemcpyAsync(&cnt, dcnt, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    *n_outliers = cnt;
    if (cnt > outlier_capacity) fail(MGRX_CAPACITY_EXCEEDED, "%llu outliers exceed capacity %llu", cnt,
                                     (unsigned long long)outlier_capacity);
    if (cnt) {
      cuda_check(cudaMemcpyAsync(h_outlier_pos, dpos, cnt * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
      cuda_check(cudaMemcpyAsync(h_outlier_val, dval, cnt * es, cudaMemcpyDeviceToHost, c->stream), "D2H");
    }
    const int rc = mgrx_gpu_encode_labels(c, dlab, uint64_t(N), h_enc, enc_capacity, enc_size);
    if (rc != MGRX_OK) fail(rc, "%s", c->last_error.c_str());
  });
}

int mgrx_gpu_field_stats(mgrx_gpu_ctx* c, int dtype, uint64_t n, const void* d_field, double* min_value,
                         double* max_value, uint64_t* first_nonfinite) {
  return guarded(c, [&] {
    if ((n && !d_field) || !min_value || !max_value || !first_nonfinite) fail(MGRX_INVALID_ARGUMENT, "null argument");
    if (dtype == MGRX_F32)
      field_stats_run<float>(c, static_cast<const float*>(d_field), int64_t(n), min_value, max_value,
                             first_nonfinite);
    else
      field_stats_run<double>(c, static_cast<const double*>(d_field), int64_t(n), min_value, max_value,
                              first_nonfinite);
  });
}

int mgrx_gpu_decompose_checked(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int stop,
                               const void* d_field, void* d_out, double* min_value, double* max_value,
                               uint64_t* first_nonfinite) {
  return guarded(c, [&] {
    if (!dims || !d_field || !d_out || !min_value || !max_value || !first_nonfinite)
      fail(MGRX_INVALID_ARGUMENT, "null argument");
    Plan* p = get_plan(c, dtype, nd, dims, levels, stop);
    const int64_t N = p->h.node[p->h.L];
    nf_arm(c);
    struct Disarm {
      mgrx_gpu_ctx* c;
      ~Disarm() { c->nf_armed = false; }
    } disarm{c};
    if (dtype == MGRX_F32)
      decompose_impl<float>(c, *p, static_cast<const float*>(d_field), static_cast<float*>(d_out), nullptr);
    else
      decompose_impl<double>(c, *p, static_cast<const double*>(d_field), static_cast<double*>(d_out), nullptr);
    unsigned flag = 0;
    double lo = INFINITY, hi = -INFINITY;
    uint64_t bad = uint64_t(N);
    if (!nf_read(c, &flag, &lo, &hi) || flag) {  // separate pass (or the exact first offset)
      if (dtype == MGRX_F32)
        field_stats_run<float>(c, static_cast<const float*>(d_field), N, &lo, &hi, &bad);
      else
        field_stats_run<double>(c, static_cast<const double*>(d_field), N, &lo, &hi, &bad);
    }
    *min_value = lo;
    *max_value = hi;
    *first_nonfinite = bad;
    if (bad < uint64_t(N))
      fail(MGRX_NONFINITE_DATA, "non-finite value at offset %llu", (unsigned long long)bad);
  });
}

int mgrx_host_compress(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, const void* h_field,
                       const double* bin_widths, int adaptive, int force_stop, const double* e_per_level,
                       const double* interp_penalty, const double* lorenzo_penalty, uint8_t* h_sections,
                       uint64_t sections_capacity, uint64_t* section_sizes, uint64_t* h_outlier_pos,
                       void* h_outlier_val, uint64_t outlier_capacity, uint64_t* n_outliers, void* h_coarse,
                       int* stop_level) {
  return guarded(c, [&] {
    if (!dims || !h_field || !bin_widths || !h_sections || !section_sizes || !n_outliers || !stop_level)
      fail(MGRX_INVALID_ARGUMENT, "null argument");
    if (adaptive && force_stop < 0 && (!e_per_level || !interp_penalty || !lorenzo_penalty))
      fail(MGRX_INVALID_ARGUMENT, "adaptive stop needs the per-level penalty tables");
    if (dtype == MGRX_F32)
      compress_core<float>(c, nd, dims, levels, static_cast<const float*>(h_field), bin_widths, adaptive, force_stop,
                           e_per_level, interp_penalty, lorenzo_penalty, h_sections, sections_capacity,
                           section_sizes, h_outlier_pos, static_cast<float*>(h_outlier_val), outlier_capacity,
                           n_outliers, static_cast<float*>(h_coarse), stop_level);
    else
      compress_core<double>(c, nd, dims, levels, static_cast<const double*>(h_field), bin_widths, adaptive,
                            force_stop, e_per_level, interp_penalty, lorenzo_penalty, h_sections, sections_capacity,
                            section_sizes, h_outlier_pos, static_cast<double*>(h_outlier_val), outlier_capacity,
                            n_outliers, static_cast<double*>(h_coarse), stop_level);
  });
}

int mgrx_host_decompose_adaptive(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels,
                                 const void* h_field, const double* e_per_level, const double* interp_penalty,
                                 const double* lorenzo_penalty, int anchor_step, int min_stop_level, void* h_out,
                                 int* stop_level) {
  return guarded(c, [&] {
    if (!dims || !h_field || !e_per_level || !interp_penalty || !lorenzo_penalty || !h_out || !stop_level)
      fail(MGRX_INVALID_ARGUMENT, "null argument");
    if (dtype == MGRX_F32)
      decompose_adaptive_impl<float>(c, nd, dims, levels, static_cast<const float*>(h_field), e_per_level,
                                     interp_penalty, lorenzo_penalty, anchor_step, min_stop_level,
                                     static_cast<float*>(h_out), stop_level);
    else
      decompose_adaptive_impl<double>(c, nd, dims, levels, static_cast<const double*>(h_field), e_per_level,
                                      interp_penalty, lorenzo_penalty, anchor_step, min_stop_level,
                                      static_cast<double*>(h_out), stop_level);
  });
}

// ---- adaptive stop decision ------------------------

int mgrx_gpu_choose_stop(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* level_dims, const void* d_block,
                         double e, const double* interp_penalty, double lorenzo_penalty, int anchor_step,
                         double* totals, int* stop) {
  return guarded(c, [&] {
    if (!level_dims || !d_block || !interp_penalty || !stop) fail(MGRX_INVALID_ARGUMENT, "null argument");
    if (nd < 1 || nd > kMaxD) fail(MGRX_INVALID_DIMS, "choose_stop: rank out of range");
    if (anchor_step < 1) fail(MGRX_INVALID_ARGUMENT, "choose_stop: anchor step must be positive");
    int64_t ext[kMaxD];
    for (int i = 0; i < nd; ++i) ext[i] = int64_t(level_dims[i]);
    const int64_t nb = stop_blocks(nd, ext, anchor_step);
    double tot[2] = {0.0, 0.0};
    if (nb == 0) {  // too small to sample: stop (choose_stop, adaptive.hpp:101)
      *stop = 1;
    } else {
      const size_t bytes = size_t(nb) * 2 * sizeof(double);
      ensure(reinterpret_cast<void**>(&c->stop_dev), &c->stop_dev_bytes, bytes, c, "cudaMalloc(stop)");
      if (c->stop_host_bytes < bytes) {
        if (c->stop_host) cudaFreeHost(c->stop_host);
        c->stop_host = nullptr;
        c->stop_host_bytes = 0;
        cuda_check(cudaMallocHost(reinterpret_cast<void**>(&c->stop_host), bytes), "cudaMallocHost(stop)");
        c->stop_host_bytes = bytes;
      }
      cudaError_t err;
      if (dtype == MGRX_F32)
        err = block_errors<float>(static_cast<const float*>(d_block), nd, ext, anchor_step, e, interp_penalty,
                                  lorenzo_penalty, c->stop_dev, exec(c));
      else
        err = block_errors<double>(static_cast<const double*>(d_block), nd, ext, anchor_step, e, interp_penalty,
                                   lorenzo_penalty, c->stop_dev, exec(c));
      cuda_check(err, "choose_stop");
      cuda_check(cudaMemcpyAsync(c->stop_host, c->stop_dev, bytes, cudaMemcpyDeviceToHost, c->stream), "D2H");
      cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
      for (int64_t b = 0; b < nb; ++b) {  // total += block, in anchor order (adaptive.hpp:77-79)
        tot[0] += c->stop_host[2 * b];
        tot[1] += c->stop_host[2 * b + 1];
      }
      *stop = tot[0] < tot[1] ? 1 : 0;
    }
    if (totals) {
      totals[0] = tot[0];
      totals[1] = tot[1];
    }
  });
}

// ---- label entropy coding --------------------------

}  // extern "C"

namespace {
// code_lengths (src/huffman.cpp:84-127): heap Huffman, the heap ordered by
// (weight, node index) like the reference's priority_queue<pair, greater>.
std::vector<int> huff_code_lengths(const std::vector<uint64_t>& freq) {
  const size_t n = freq.size();
  std::vector<int64_t> parent;
  std::vector<int64_t> node_of(n, -1);
  using Item = std::pair<uint64_t, size_t>;
  std::priority_queue<Item, std::vector<Item>, std::greater<Item>> heap;
  for (size_t s = 0; s < n; ++s)
    if (freq[s]) {
      node_of[s] = int64_t(parent.size());
      heap.emplace(freq[s], parent.size());
      parent.push_back(-1);
    }
  std::vector<int> lens(n, 0);
  if (parent.empty()) return lens;
  if (parent.size() == 1) {
    for (size_t s = 0; s < n; ++s)
      if (node_of[s] >= 0) lens[s] = 1;
    return lens;
  }
  while (heap.size() > 1) {
    const Item a = heap.top();
    heap.pop();
    const Item b = heap.top();
    heap.pop();
    const size_t node = parent.size();
    parent.push_back(-1);
    parent[a.second] = int64_t(node);
    parent[b.second] = int64_t(node);
    heap.emplace(a.first + b.first, node);
  }
  for (size_t s = 0; s < n; ++s) {
    int64_t v = node_of[s];
    if (v < 0) continue;
    int len = 0;
    while (parent[size_t(v)] >= 0) {
      v = parent[size_t(v)];
      ++len;
    }
    lens[s] = len;
  }
  return lens;
}

// canonicalize (:138-160) + the per-symbol reversed codes of encode_labels
// (:228-236), packed as (reversed code << 6) | length.
std::vector<unsigned long long> huff_codes(const std::vector<int>& lens) {
  int max_len = 0;
  for (int l : lens) max_len = std::max(max_len, l);
  std::vector<unsigned long long> code(lens.size(), 0);
  if (max_len == 0) return code;
  if (max_len > 57) fail(MGRX_INVALID_INPUT, "code length too large");
  std::vector<uint64_t> count(size_t(max_len) + 1, 0), first(size_t(max_len) + 1, 0);
  for (int l : lens)
    if (l > 0) ++count[size_t(l)];
  uint64_t c = 0;
  for (int l = 1; l <= max_len; ++l) {
    c <<= 1;
    first[size_t(l)] = c;
    c += count[size_t(l)];
  }
  // canonical order: by length, then by symbol value
  for (int l = 1; l <= max_len; ++l)
    for (size_t s = 0; s < lens.size(); ++s)
      if (lens[s] == l) {
        const uint64_t cw = first[size_t(l)]++;
        uint64_t r = 0;
        for (int i = 0; i < l; ++i) r |= ((cw >> i) & 1ull) << (l - 1 - i);
        code[s] = (r << 6) | uint64_t(l);
      }
  return code;
}

void put_le(uint8_t* p, uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) p[i] = uint8_t(v >> (8 * i));
}
}  // namespace

extern "C" {

int mgrx_gpu_encode_labels(mgrx_gpu_ctx* c, const int32_t* d_labels, uint64_t n, uint8_t* h_out, uint64_t capacity,
                           uint64_t* out_size) {
  return guarded(c, [&] {
    if (!out_size || (n && !d_labels)) fail(MGRX_INVALID_ARGUMENT, "null argument");
    if (n == 0) {  // min, range, bit count (huffman.cpp:211-216)
      *out_size = 16;
      if (capacity < 16 || !h_out) fail(MGRX_CAPACITY_EXCEEDED, "output capacity %llu < 16", (unsigned long long)capacity);
      std::memset(h_out, 0, 16);
      return;
    }
    const Exec ex = exec(c);
    struct Dev {
      mgrx_gpu_ctx* c;
      std::vector<void*> p;
      void* get(size_t bytes) {
        void* q = nullptr;
        cuda_check(cudaMallocAsync(&q, bytes, c->stream), "cudaMallocAsync");
        p.push_back(q);
        return q;
      }
      ~Dev() {
        for (void* q : p) cudaFreeAsync(q, c->stream);
      }
    } dev{c, {}};
    int* d_mm = static_cast<int*>(dev.get(8));
    cuda_check(label_minmax(d_labels, int64_t(n), d_mm, ex), "label min/max");
    int mm[2];
    cuda_check(cudaMemcpyAsync(mm, d_mm, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
    const int lo = mm[0];
    const int64_t range = int64_t(mm[1]) - lo + 1;
    if (range > (int64_t(1) << 17)) fail(MGRX_INVALID_INPUT, "label alphabet too large");
    auto* d_freq = static_cast<unsigned long long*>(dev.get(size_t(range) * 8));
    cuda_check(label_hist(d_labels, int64_t(n), lo, int(range), d_freq, ex), "label histogram");
    std::vector<uint64_t> freq(static_cast<size_t>(range));
    cuda_check(cudaMemcpyAsync(freq.data(), d_freq, size_t(range) * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
    const std::vector<int> lens = huff_code_lengths(freq);
    const std::vector<unsigned long long> code = huff_codes(lens);
    uint64_t nbits = 0;
    for (size_t s = 0; s < freq.size(); ++s) nbits += freq[s] * uint64_t(lens[s]);
    const uint64_t hdr = 8 + uint64_t(range) + 8, payload = (nbits + 7) / 8;
    *out_size = hdr + payload;
    if (!h_out || capacity < *out_size)
      fail(MGRX_CAPACITY_EXCEEDED, "output capacity %llu < %llu", (unsigned long long)capacity,
           (unsigned long long)*out_size);
    auto* d_code = static_cast<unsigned long long*>(dev.get(size_t(range) * 8));
    cuda_check(cudaMemcpyAsync(d_code, code.data(), size_t(range) * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
    const int64_t nch = enc_chunks(int64_t(n));
    auto* d_cb = static_cast<unsigned long long*>(dev.get(size_t(nch) * 8));
    cuda_check(label_chunk_bits(d_labels, int64_t(n), lo, d_code, d_cb, ex), "chunk bits");
    std::vector<unsigned long long> cb(static_cast<size_t>(nch));
    cuda_check(cudaMemcpyAsync(cb.data(), d_cb, size_t(nch) * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
    unsigned long long acc = 0;
    for (auto& v : cb) {  // exclusive scan of the chunks' bits
      const unsigned long long t = v;
      v = acc;
      acc += t;
    }
    if (acc != nbits) fail(MGRX_CUDA_ERROR, "encode: bit count mismatch");
    cuda_check(cudaMemcpyAsync(d_cb, cb.data(), size_t(nch) * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
    const uint64_t nwords = nbits / 64 + 2;
    auto* d_words = static_cast<unsigned long long*>(dev.get(size_t(nwords) * 8));
    cuda_check(label_emit(d_labels, int64_t(n), lo, d_code, d_cb, d_words, nwords, ex), "emit");
    put_le(h_out, uint32_t(lo), 4);
    put_le(h_out + 4, uint64_t(range), 4);
    for (int64_t s = 0; s < range; ++s) h_out[8 + s] = uint8_t(lens[size_t(s)]);
    put_le(h_out + 8 + range, nbits, 8);
    if (payload)
      cuda_check(cudaMemcpyAsync(h_out + hdr, d_words, size_t(payload), cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
  });
}

// ---- slab mode ------------------------------------------

namespace {
// The plan of the full field (stop 0) and its fused level `level`.
Plan* slab_plan(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int level) {
  if (!dims) fail(MGRX_INVALID_ARGUMENT, "null argument");
  Plan* p = get_plan(c, dtype, nd, dims, levels, 0);
  if (level < 1 || level > p->h.L) fail(MGRX_INVALID_LEVEL, "slab: level out of range");
  if (!p->fused[level].enabled) fail(MGRX_INVALID_ARGUMENT, "slab: level is not on the fused 3-D path");
  return p;
}
}  // namespace

int mgrx_gpu_slab_level(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int level,
                        int64_t* info) {
  return guarded(c, [&] {
    if (!dims || !info) fail(MGRX_INVALID_ARGUMENT, "null argument");
    Plan* p = get_plan(c, dtype, nd, dims, levels, 0);
    if (level < 1 || level > p->h.L) fail(MGRX_INVALID_LEVEL, "slab: level out of range");
    const Fused3DPlan& fp = p->fused[level];
    const LevelGeom& g = p->geom[level];
    for (int i = 0; i < 3; ++i) {
      info[i] = i < g.d ? g.n[i] : 1;
      info[3 + i] = i < g.d ? g.m[i] : 1;
    }
    info[6] = (fp.enabled && c->path == 0) ? 1 : 0;
    info[7] = int64_t(p->h.node[level - 1]);
    info[8] = int64_t(p->h.node[level]);
  });
}

int mgrx_gpu_slab_dec_plane(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int level,
                            uint64_t k0, uint64_t k1, const void* d_blk, void* d_out, void* d_coarse, double* d_G,
                            int64_t odd_shift) {
  return guarded(c, [&] {
    if (!d_blk || !d_out || !d_coarse || !d_G) fail(MGRX_INVALID_ARGUMENT, "null argument");
    Plan* p = slab_plan(c, dtype, nd, dims, levels, level);
    const size_t off = p->h.node[level - 1];
    Fused3DPlan fp = p->fused[level];
    fp.g.odd_shift = odd_shift;
    cudaError_t e;
    if (dtype == MGRX_F32)
      e = fused3d_slab_dec_plane<float>(static_cast<const float*>(d_blk), static_cast<float*>(d_out) + off,
                                        static_cast<float*>(d_coarse), d_G, fp, int64_t(k0), int64_t(k1),
                                        exec(c, level));
    else
      e = fused3d_slab_dec_plane<double>(static_cast<const double*>(d_blk), static_cast<double*>(d_out) + off,
                                         static_cast<double*>(d_coarse), d_G, fp, int64_t(k0),
                                         int64_t(k1), exec(c, level));
    cuda_check(e, "slab dec plane");
  });
}

int mgrx_gpu_slab_rec_plane(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int level,
                            uint64_t k0, uint64_t k1, const void* d_coeffs, double* d_G, int64_t odd_shift) {
  return guarded(c, [&] {
    if (!d_coeffs || !d_G) fail(MGRX_INVALID_ARGUMENT, "null argument");
    Plan* p = slab_plan(c, dtype, nd, dims, levels, level);
    const size_t off = p->h.node[level - 1];
    Fused3DPlan fp = p->fused[level];
    fp.g.odd_shift = odd_shift;
    cudaError_t e;
    if (dtype == MGRX_F32)
      e = fused3d_slab_rec_plane<float>(static_cast<const float*>(d_coeffs) + off, d_G, fp, int64_t(k0),
                                        int64_t(k1), exec(c, level));
    else
      e = fused3d_slab_rec_plane<double>(static_cast<const double*>(d_coeffs) + off, d_G, fp,
                                         int64_t(k0), int64_t(k1), exec(c, level));
    cuda_check(e, "slab rec plane");
  });
}

int mgrx_gpu_slab_inplane(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int level,
                          uint64_t k0, uint64_t k1, double* d_G) {
  return guarded(c, [&] {
    if (!d_G) fail(MGRX_INVALID_ARGUMENT, "null argument");
    Plan* p = slab_plan(c, dtype, nd, dims, levels, level);
    cuda_check(fused3d_slab_inplane(d_G, p->fused[level], p->thomas[level], int64_t(k0), int64_t(k1), exec(c, level)),
               "slab in-plane solves");
  });
}

int mgrx_gpu_slab_axis0(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int level,
                        uint64_t width, double* d_Gt) {
  return guarded(c, [&] {
    if (!d_Gt) fail(MGRX_INVALID_ARGUMENT, "null argument");
    Plan* p = slab_plan(c, dtype, nd, dims, levels, level);
    cuda_check(fused3d_slab_axis0(d_Gt, int64_t(width), p->fused[level], p->thomas[level], exec(c, level)),
               "slab axis-0 solve");
  });
}

int mgrx_gpu_slab_apply(mgrx_gpu_ctx* c, int dtype, void* d_coarse, const double* d_z, uint64_t n, double sign) {
  return guarded(c, [&] {
    if (!d_coarse || !d_z) fail(MGRX_INVALID_ARGUMENT, "null argument");
    cudaError_t e;
    if (dtype == MGRX_F32)
      e = apply_correction<float>(static_cast<float*>(d_coarse), d_z, int64_t(n), sign, exec(c));
    else
      e = apply_correction<double>(static_cast<double*>(d_coarse), d_z, int64_t(n), sign, exec(c));
    cuda_check(e, "slab apply");
  });
}

int mgrx_gpu_slab_interp(mgrx_gpu_ctx* c, int dtype, int nd, const uint64_t* dims, int levels, int level,
                         uint64_t p0, uint64_t p1, const void* d_coeffs, const void* d_coarse, void* d_fine,
                         int64_t odd_shift) {
  return guarded(c, [&] {
    if (!d_coeffs || !d_coarse || !d_fine) fail(MGRX_INVALID_ARGUMENT, "null argument");
    Plan* p = slab_plan(c, dtype, nd, dims, levels, level);
    const size_t off = p->h.node[level - 1];
    Fused3DPlan fp = p->fused[level];
    fp.g.odd_shift = odd_shift;
    cudaError_t e;
    if (dtype == MGRX_F32)
      e = fused3d_slab_interp<float>(static_cast<const float*>(d_coeffs) + off, static_cast<const float*>(d_coarse),
                                     static_cast<float*>(d_fine), fp, int64_t(p0), int64_t(p1),
                                     exec(c, level));
    else
      e = fused3d_slab_interp<double>(static_cast<const double*>(d_coeffs) + off, static_cast<const double*>(d_coarse),
                                      static_cast<double*>(d_fine), fp, int64_t(p0), int64_t(p1),
                                      exec(c, level));
    cuda_check(e, "slab interpolation");
  });
}

int mgrx_gpu_slab_pack(mgrx_gpu_ctx* c, const double* d_src, uint64_t rows, uint64_t pitch, const uint64_t* cb,
                       int nparts, double* d_dst) {
  return guarded(c, [&] {
    if (!d_src || !d_dst || !cb || nparts <= 0 || nparts > 256) fail(MGRX_INVALID_ARGUMENT, "bad pack arguments");
    cuda_check(slab_pack(d_src, int64_t(rows), int64_t(pitch), cb, nparts, d_dst, false, exec(c)), "slab pack");
  });
}

int mgrx_gpu_slab_unpack(mgrx_gpu_ctx* c, const double* d_src, uint64_t rows, uint64_t pitch, const uint64_t* cb,
                         int nparts, double* d_dst) {
  return guarded(c, [&] {
    if (!d_src || !d_dst || !cb || nparts <= 0 || nparts > 256) fail(MGRX_INVALID_ARGUMENT, "bad unpack arguments");
    cuda_check(slab_pack(d_src, int64_t(rows), int64_t(pitch), cb, nparts, d_dst, true, exec(c)), "slab unpack");
  });
}

}  // extern "C"
