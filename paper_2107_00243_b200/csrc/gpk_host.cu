// Host driver and C-ABI of libgpkrylov_cuda.so.
//
// Mirrors the reference's C++ interface (proj/include/gpkrylov):
//   KernelOperator (kernels.hpp:157-336)      -> gpk_set_data / gpk_set_params / gpk_kernel_*
//   pcg_solve / batched_pcg (krylov.hpp)      -> mbcg() : one batched CG over all columns
//   DiagPlusLowRank + pivoted_cholesky (+deriv factors) (preconditioners.hpp) -> Precond
//   slq_quadrature / vr_logdet / trace_residual (trace_estimation.hpp) -> host SLQ + fused passes
//   evaluate_mll (gp_likelihood.hpp:51-103)  -> evaluate()
// The heavy lifting runs in the sm_100a kernels (gpk_mvm*.cu, gpk_deriv.cu,
// gpk_linalg.cu); this file owns the control flow, O(m^2) tridiagonal
// eigen-solves, O(k^3) inner Cholesky and error mapping.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "gpk_internal.h"
#include "gpk_linalg.h"
#include "gpkrylov_cuda.h"

namespace {

struct GpkError {
  gpk_status code;
  std::string msg;
};
[[noreturn]] void fail(gpk_status c, const std::string& m) { throw GpkError{c, m}; }
void require(bool c, const std::string& m) {
  if (!c) fail(GPK_INPUT_ERROR, m);
}

#define CB(x)                                                                            \
  do {                                                                                   \
    cublasStatus_t s_ = (x);                                                             \
    if (s_ != CUBLAS_STATUS_SUCCESS) fail(GPK_CUDA_ERROR, std::string(#x) + ": cuBLAS status " + std::to_string(s_)); \
  } while (0)
#define CS(x)                                                                            \
  do {                                                                                   \
    cusolverStatus_t s_ = (x);                                                           \
    if (s_ != CUSOLVER_STATUS_SUCCESS) fail(GPK_CUDA_ERROR, std::string(#x) + ": cuSOLVER status " + std::to_string(s_)); \
  } while (0)
#define CK(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) fail(GPK_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Device buffers come from the stream-ordered pool allocator on the context's
// stream (pool release threshold = max): scratch allocated and freed inside a
// call is recycled without any device synchronisation.
thread_local cudaStream_t tl_stream = nullptr;

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;
  cudaStream_t s = nullptr;
  void ensure(size_t cnt) {
    if (cnt == 0) cnt = 1;
    if (cnt <= cap) return;
    release();
    s = tl_stream;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&p), cnt * sizeof(T), s));
    cap = cnt;
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    cap = 0;
  }
  ~DBuf() { release(); }
};

std::string num(double v) { return std::to_string(v); }  // the reference formats with std::to_string

// ---------------------------------------------------------------------------
// Tridiagonal eigen-solve for SLQ (trace_estimation.hpp:88-110): implicit QL
// with Wilkinson-type shifts, tracking only the first row of the eigenvector
// matrix (the quadrature weights), O(m^2).
// ---------------------------------------------------------------------------
bool tridiag_eig_first_row(std::vector<double>& d, std::vector<double> e, std::vector<double>& z0) {
  const int m = static_cast<int>(d.size());
  z0.assign(m, 0.0);
  if (m == 0) return true;
  z0[0] = 1.0;
  e.resize(m, 0.0);
  e[m - 1] = 0.0;
  for (int l = 0; l < m; ++l) {
    int iter = 0, mm;
    do {
      for (mm = l; mm < m - 1; ++mm) {
        const double dd = std::fabs(d[mm]) + std::fabs(d[mm + 1]);
        if (std::fabs(e[mm]) <= 2.220446049250313e-16 * dd) break;
      }
      if (mm != l) {
        if (++iter > 60) return false;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = d[mm] - d[l] + e[l] / (g + (g >= 0.0 ? r : -r));
        double s = 1.0, c = 1.0, p = 0.0;
        bool deflated = false;
        for (int i = mm - 1; i >= l; --i) {
          const double f = s * e[i];
          const double b = c * e[i];
          r = std::hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[mm] = 0.0;
            deflated = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          const double zf = z0[i + 1];
          z0[i + 1] = s * z0[i] + c * zf;
          z0[i] = c * z0[i] - s * zf;
        }
        if (deflated) continue;
        d[l] -= p;
        e[l] = g;
        e[mm] = 0.0;
      }
    } while (mm != l);
  }
  return true;
}

struct SlqOut {
  double value = 0.0;
  int clamped = 0;
};
SlqOut slq_log(const std::vector<double>& diag, const std::vector<double>& sub) {
  SlqOut o;
  if (diag.empty()) return o;
  std::vector<double> d = diag, z0;
  if (!tridiag_eig_first_row(d, sub, z0)) fail(GPK_NUMERICAL_ERROR, "slq_quadrature: eigensolver failed");
  double amax = 0.0;
  for (double v : d) amax = std::max(amax, std::fabs(v));
  const double floor_value = 1e-12 * amax;
  for (size_t j = 0; j < d.size(); ++j) {
    double node = d[j];
    if (node < floor_value) {
      node = floor_value;
      ++o.clamped;
    }
    o.value += (z0[j] * z0[j]) * std::log(node);
  }
  return o;
}

double unbiased_variance(const std::vector<double>& v) {
  if (v.size() < 2) return 0.0;
  double mean = 0.0;
  for (double x : v) mean += x;
  mean /= static_cast<double>(v.size());
  double ss = 0.0;
  for (double x : v) ss += (x - mean) * (x - mean);
  return ss / static_cast<double>(v.size() - 1);
}

// ---------------------------------------------------------------------------
// small kernels local to the driver
// ---------------------------------------------------------------------------
template <typename T>
__global__ void to_padded_kernel(const double* __restrict__ src, long long lds, int n, int n_pad, int t,
                                 T* __restrict__ dst) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(t) * n_pad) return;
  const int c = static_cast<int>(idx / n_pad), i = static_cast<int>(idx % n_pad);
  dst[idx] = static_cast<T>(i < n ? src[c * lds + i] : 0.0);
}
// t_{w,i} = (dL_w' q_i).(L' z_i) + (L' q_i).(dL_w' z_i)  (LowRankDerivOp::apply,
// preconditioners.hpp:62-69): one warp per (w, i), lane-strided sums + a fixed butterfly
__global__ void precond_trace_terms_kernel(const double* __restrict__ Bq, const double* __restrict__ Bz,
                                           const double* __restrict__ A, int k, int kw, int l, int nw,
                                           double* __restrict__ out) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (gw >= nw * l) return;
  const int w = gw / l, i = gw % l;
  const double* bq = Bq + static_cast<size_t>(i) * kw + static_cast<size_t>(w) * k;
  const double* bz = Bz + static_cast<size_t>(i) * kw + static_cast<size_t>(w) * k;
  const double* aq = A + static_cast<size_t>(i) * k;
  const double* az = A + static_cast<size_t>(l + i) * k;
  double acc = 0.0;
  for (int q = lane; q < k; q += 32) acc += bq[q] * az[q] + aq[q] * bz[q];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[static_cast<size_t>(w) * l + i] = acc;
}
__global__ void gather_slots_kernel(const gpk::SlotState* __restrict__ src, const int* __restrict__ map, int nt,
                                    gpk::SlotState* __restrict__ dst) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < nt) dst[q] = src[map[q]];
}
// page-locked host memory (the pipelined CG state read-back and the small uploads of the
// compaction maps must not drain the stream)
struct Pinned {
  char* p = nullptr;
  size_t cap = 0;
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    if (cudaMallocHost(reinterpret_cast<void**>(&p), bytes) != cudaSuccess) {
      p = nullptr;
      fail(GPK_CUDA_ERROR, "cudaMallocHost failed");
    }
    cap = bytes;
  }
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
};
struct EventPair {
  cudaEvent_t e[2] = {nullptr, nullptr};
  cudaEvent_t get(int i) {
    if (!e[i]) CK(cudaEventCreateWithFlags(&e[i], cudaEventDisableTiming));
    return e[i];
  }
  ~EventPair() {
    for (auto x : e)
      if (x) cudaEventDestroy(x);
  }
};
__global__ void add_diag_kernel(double* __restrict__ a, int k, double v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) a[static_cast<long long>(i) * (k + 1)] += v;
}
__global__ void fill_kernel(double* __restrict__ p, long long cnt, double v) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i < cnt) p[i] = v;
}
__global__ void residual_kernel(const double* __restrict__ B, long long ldb, const double* __restrict__ KX,
                                const double* __restrict__ X, double sig2, int n, long long ldn,
                                double* __restrict__ R) {
  const int s = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long o = s * ldn + i;
  R[o] = B[s * ldb + i] - (KX[o] + sig2 * X[o]);
}

// rank-order sum of world partial vectors: out[i] = sum_r parts[r * count + i]
__global__ void rank_sum_kernel(const double* __restrict__ parts, int world, long long count,
                                double* __restrict__ out) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int r = 0; r < world; ++r) s += parts[r * count + i];
  out[i] = s;
}
// full[c][r0_r + i] = gathered[r][c][i] for i < rows_r (the all-gathered row shards, padded to nmax)
__global__ void unshard_cols_kernel(const double* __restrict__ g, int world, int t, long long nmax,
                                    const int* __restrict__ r0s, const int* __restrict__ rows, double* __restrict__ full,
                                    long long ldf) {
  const int c = blockIdx.y;
  const int r = blockIdx.z;
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= rows[r]) return;
  full[c * ldf + r0s[r] + i] = g[(static_cast<long long>(r) * t + c) * nmax + i];
}

// ---------------------------------------------------------------------------
// Communicators for row sharding (one rank per GPU).  Collectives used by the
// mBCG path: all-gather of equal-size device buffers; sums are built from it
// in rank order, so every rank and every run gets bitwise the same result.
// ---------------------------------------------------------------------------
struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
};

struct NcclComm : Comm {
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c) ncclCommDestroy(c);
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    const ncclResult_t r = ncclAllGather(send, recv, bytes, ncclChar, c, st);
    if (r != ncclSuccess) fail(GPK_NCCL_ERROR, std::string("ncclAllGather: ") + ncclGetErrorString(r));
  }
};

}  // namespace

// In-process rank group (one host thread per rank, any devices): host-staged
// collectives with a generation barrier.  Used to run and test the sharded path
// on a single GPU; kernels never wait on each other, only host threads do.
struct gpk_group {
  int world = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<std::vector<char>> host;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

namespace {
struct GroupComm : Comm {
  gpk_group* g = nullptr;
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    std::vector<char>& mine = g->host[rank];
    mine.resize(bytes);
    CK(cudaMemcpyAsync(mine.data(), send, bytes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    g->barrier();
    for (int r = 0; r < world; ++r)
      CK(cudaMemcpyAsync(static_cast<char*>(recv) + r * bytes, g->host[r].data(), bytes, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    g->barrier();
  }
};

// contiguous row shards in units of 128 rows (fused-MVM row blocks never straddle ranks)
void shard_of(int n, int rank, int world, int* r0, int* r1) {
  const int nb = (n + 127) / 128;
  const int base = nb / world, extra = nb % world;
  const int b0 = rank * base + std::min(rank, extra);
  const int b1 = b0 + base + (rank < extra ? 1 : 0);
  *r0 = std::min(n, b0 * 128);
  *r1 = std::min(n, b1 * 128);
}
}  // namespace

// ===========================================================================
struct gpk_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  std::string err;
  long long launches = 0;

  // ---- data (kernels.hpp:159-173)
  int n = 0, d = 0, n_pad = 0, dp = 0;
  long long ldn = 0;  // leading dimension of the (local) n-length CG state

  // ---- row sharding: this rank owns rows [r0, r1) (nl = r1 - r0) of every
  // n-length CG / probe array; X, L, C, dL are replicated.  world == 1: r0 = 0, nl = n.
  std::unique_ptr<Comm> comm;
  int rank = 0, world = 1, r0 = 0, r1 = 0, nl = 0;
  std::vector<int> all_r0, all_rows;
  DBuf<int> d_r0, d_rows;
  DBuf<double> w_send, w_recv, w_full, w_red;

  void set_shard() {
    all_r0.assign(world, 0);
    all_rows.assign(world, 0);
    for (int r = 0; r < world; ++r) {
      int a, b;
      shard_of(n, r, world, &a, &b);
      all_r0[r] = a;
      all_rows[r] = b - a;
    }
    r0 = all_r0[rank];
    nl = all_rows[rank];
    r1 = r0 + nl;
    require(nl > 0, "gpkrylov_cuda: n too small for the number of ranks (each rank needs >= 1 row)");
    ldn = (nl + 31) / 32 * 32;
    if (world > 1) {
      d_r0.ensure(world);
      d_rows.ensure(world);
      h2d(d_r0.p, all_r0.data(), sizeof(int) * world);
      h2d(d_rows.p, all_rows.data(), sizeof(int) * world);
    }
  }
  // full[c][*] (ld ldf, all n rows) <- every rank's local rows loc[c][*] (ld ldl)
  void allgather_cols(const double* loc, long long ldl, int t, double* full, long long ldf) {
    const long long nmax = *std::max_element(all_rows.begin(), all_rows.end());
    w_send.ensure(static_cast<size_t>(t) * nmax);
    w_recv.ensure(static_cast<size_t>(world) * t * nmax);
    check_launch(gpk::launch_gather_cols(loc, ldl, nullptr, 1.0, nl, t, w_send.p, nmax, st), 1, "gather");
    comm->allgather(w_send.p, w_recv.p, sizeof(double) * static_cast<size_t>(t) * nmax, st);
    dim3 g(static_cast<unsigned>((nmax + 255) / 256), t, world);
    unshard_cols_kernel<<<g, 256, 0, st>>>(w_recv.p, world, t, nmax, d_r0.p, d_rows.p, full, ldf);
    check_launch(cudaGetLastError(), 1, "unshard");
  }
  // in-place rank-ordered sum over ranks of a device vector
  void allreduce_sum(double* buf, long long count) {
    if (world == 1 || count <= 0) return;
    w_red.ensure(static_cast<size_t>(world) * count);
    comm->allgather(buf, w_red.p, sizeof(double) * static_cast<size_t>(count), st);
    rank_sum_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, st>>>(w_red.p, world, count, buf);
    check_launch(cudaGetLastError(), 1, "rank_sum");
  }
  std::vector<double> allreduce_host(std::vector<double> v) {
    if (world == 1 || v.empty()) return v;
    DBuf<double> b;
    b.ensure(v.size());
    h2d(b.p, v.data(), sizeof(double) * v.size());
    allreduce_sum(b.p, static_cast<long long>(v.size()));
    d2h(v.data(), b.p, sizeof(double) * v.size());
    return v;
  }
  // the full (all-row) view of a local column block: the block itself on one rank
  const double* full_cols(const double* loc, long long ldl, int t, long long* ldf) {
    if (world == 1) {
      *ldf = ldl;
      return loc;
    }
    w_full.ensure(static_cast<size_t>(t) * n);
    allgather_cols(loc, ldl, t, w_full.p, n);
    *ldf = n;
    return w_full.p;
  }
  bool have_data = false, have_params = false;
  DBuf<double> X, sx, sq, ls_dev, X64s;
  DBuf<float> X32;
  // ---- params
  int family = 0;
  double log_o = 0, log_noise = 0, o = 1, o2 = 1, noise = 1e-2;
  std::vector<double> log_ls, ls;
  bool packed = false;

  // ---- preconditioner
  int pkind = 0;  // 0 none, 1 identity, 2 diag-plus-low-rank
  int k = 0;
  double pnoise = 0.0, plogdet = 0.0;
  DBuf<double> L, C, dL;
  // L, C, dL storage: unsharded, all n rows (leading dimension n); row-sharded (world > 1),
  // the own rows [r0, r1) followed by the k pivot rows (leading dimension nl + k) -- the
  // preconditioner is built and stored per rank, never replicated
  bool pshard = false;
  long long ldP = 0;
  double* Lloc() const { return pshard ? L.p : L.p + r0; }
  double* Cloc() const { return pshard ? C.p : C.p + r0; }
  double* dLloc() const { return pshard ? dL.p : dL.p + r0; }
  std::vector<long long> pivots;
  bool have_dl = false;
  std::vector<double> trace_det;  // tr(P^-1 dP_w), w = 0..d+1

  // ---- workspaces
  DBuf<double> w_part, w_y, w_kx, w_g1, w_W, w_T, w_B, w_tmp, w_tmp2, w_ps, w_hist;
  DBuf<double> st_X[2], st_R[2], st_P[2], st_Z;
  DBuf<float> w_v32, w_f32, w_vhi, w_vlo;
  bool use_tc = false;  // GPK_PREC_TF32X3: value MVMs on the tcgen05 tensor cores
  // split-K partials of the last tcgen05 MVM left unreduced for a fused consumer (the CG loop's
  // p'Ap kernel): set defer_reduce before apply_kernel, read and clear pend after
  struct PendingSplits {
    const double* part = nullptr;
    int splits = 0;
    long long sstride = 0, ldp = 0;
  } pend;
  bool defer_reduce = false;
  bool fuse_reduce = [] {  // env GPK_FUSE_REDUCE=0: separate reduce_splits launch (A/B)
    const char* e = std::getenv("GPK_FUSE_REDUCE");
    return !(e && e[0] == '0');
  }();
  bool vmax_ready = false;  // w_vmax holds the column maxima of the next direction block
  bool use_fused_cg = [] {  // env GPK_FUSED_CG=0 selects the unfused per-step kernels (A/B checks)
    const char* e = std::getenv("GPK_FUSED_CG");
    return !(e && std::atoi(e) == 0);
  }();
  DBuf<unsigned> w_cnt, w_cnt2;
  DBuf<double> w_prz, w_pzz;
  bool use_f64g = [] {  // env GPK_F64G=0 selects the FP64-pipe fp64 MVM (A/B checks)
    const char* e = std::getenv("GPK_F64G");
    return !(e && std::atoi(e) == 0);
  }();
  bool use_wood_s = [] {  // env GPK_WOOD=0 selects the unstaged g1/g2 Woodbury kernels (A/B checks)
    const char* e = std::getenv("GPK_WOOD");
    return !(e && std::atoi(e) == 0);
  }();
  // the single-rank vector phase as one cooperative launch (env GPK_COOP=0: the five-launch path)
  bool use_coop = gpk::cg_iter_coop_available();
  DBuf<double> w_ppap;
  bool use_persistent_pchol = [] {  // env GPK_PCHOL_STEPS=1 selects the per-step kernels (A/B checks)
    const char* e = std::getenv("GPK_PCHOL_STEPS");
    return !(e && std::atoi(e) == 1);
  }();
  // Pipelined CG state read-back (env GPK_PIPE=0 disables): the slot states of iteration
  // it are copied to pinned memory asynchronously and examined after iteration it + 1 has
  // been enqueued, so the device never idles on the host round trip.  Converged columns are
  // frozen on the device (flag), so the one-iteration-late decision changes no result.
  bool use_pipe = [] {
    const char* e = std::getenv("GPK_PIPE");
    return !(e && std::atoi(e) == 0);
  }();
  Pinned snap_h, ring_h;
  size_t ring_off = 0;
  EventPair snap_ev;
  // upload through a pinned ring (stream-ordered, no drain); wraps after a stream sync
  void h2d_ring(void* dst, const void* src, size_t bytes) {
    constexpr size_t cap = 1 << 20;
    ring_h.ensure(cap);
    const size_t b = (bytes + 255) & ~static_cast<size_t>(255);
    if (b > cap) {
      h2d(dst, src, bytes);
      sync();
      return;
    }
    if (ring_off + b > cap) {
      sync();
      ring_off = 0;
    }
    std::memcpy(ring_h.p + ring_off, src, bytes);
    CK(cudaMemcpyAsync(dst, ring_h.p + ring_off, bytes, cudaMemcpyHostToDevice, st));
    ring_off += b;
  }
  int sync_every = [] {  // CG iterations between host round trips (env GPK_SYNC_EVERY, default 1:
    const char* e = std::getenv("GPK_SYNC_EVERY");  // measured no gain from lazier syncs at C2)
    const int v = e ? std::atoi(e) : 1;
    return v >= 1 && v <= 64 ? v : 1;
  }();
  // persistent Gram/direct tcgen05 MVM (env GPK_TCG_PERSIST=0: one CTA per (row block, split) unit)
  int tcg_ctas = [] {
    const char* e = std::getenv("GPK_TCG_PERSIST");
    if (e && std::atoi(e) == 0) return 0;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return 0;
    return sms;
  }();
  int tcg_unit_order = [] {  // env GPK_TCG_ORDER=0/1 forces the unit order (A/B); default: by operand footprint
    const char* e = std::getenv("GPK_TCG_ORDER");
    return e ? std::atoi(e) : -1;
  }();
  // TEST HOOK (env GPK_TCG_CTAS=c): cap the persistent MVM grid at c CTAs without changing the
  // unit decomposition (splits_for_tcg keeps the SM count), so every CTA runs several units --
  // row-block changes and same-row split changes -- with results bitwise those of the full grid
  int tcg_grid_cap = [] {
    const char* e = std::getenv("GPK_TCG_CTAS");
    const int v = e ? std::atoi(e) : 0;
    return v > 0 ? v : 0;
  }();
  int tc_flush = [] {   // j-tiles per TMEM accumulation group (env GPK_TC_FLUSH, default 2)
    const char* e = std::getenv("GPK_TC_FLUSH");
    const int v = e ? std::atoi(e) : 2;
    return v >= 1 && v <= 8 ? v : 2;
  }();
  // Gram-variant tensor-core MVM (gpk_mvm_tcg.cuh): packed centred coordinates + norms
  int mvm_variant = [] {  // GPK_MVM_AUTO / DIRECT / GRAM (env GPK_MVM_VARIANT, default auto)
    const char* e = std::getenv("GPK_MVM_VARIANT");
    const int v = e ? std::atoi(e) : 0;
    return v >= 0 && v <= 2 ? v : 0;
  }();
  bool gram_ok = false;   // the value MVMs of the tf32x3 path use the Gram kernel
  bool tcg_direct = false;  // ... or the same tcgen05 pipeline with direct-difference distances (d <= 8)
  float gram_maxnorm = 0.0f;
  DBuf<float> Xgh, Xgl, Xgn;
  DBuf<double> Xgmu;
  DBuf<uint16_t> w_h16hi, w_h16lo;  // fp16 V tiles of the Gram variant
  DBuf<unsigned long long> w_vmax;
  DBuf<double> w_colscale;
  DBuf<double> w_v64, w_f64;
  DBuf<gpk::SlotState> w_ss[2];
  DBuf<int> w_map;
  DBuf<double> w_argval;
  DBuf<long long> w_argidx;

  // ---- telemetry
  long long entries = 0, flops = 0;
  struct Prof {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
    std::vector<double> pflops, pentries;
    double ms = 0.0, fl = 0.0, en = 0.0;
    long long launches = 0;
  };
  bool prof_on = false;
  unsigned prof_mask = 3u;  // kinds recorded while enabled (bit k = kind k)
  Prof prof[4];  // 0: reduced-precision value MVM, 1: derivative pass, 2: fp64 MVM, 3: CG vector phase
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t ev_get() {
    if (!ev_pool.empty()) {
      cudaEvent_t e = ev_pool.back();
      ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
  }
  // bracket one launch of kind `kd` with events when profiling is on
  std::pair<cudaEvent_t, cudaEvent_t> prof_begin(int kd) {
    if (!prof_on || !(prof_mask & (1u << kd))) return {nullptr, nullptr};
    cudaEvent_t a = ev_get(), b = ev_get();
    CK(cudaEventRecord(a, st));
    return {a, b};
  }
  void prof_end(int kd, std::pair<cudaEvent_t, cudaEvent_t> ev, double fl, double en) {
    if (!ev.first) return;
    CK(cudaEventRecord(ev.second, st));
    prof[kd].pending.push_back(ev);
    prof[kd].pflops.push_back(fl);
    prof[kd].pentries.push_back(en);
  }
  void prof_collect() {
    for (auto& p : prof) {
      if (p.pending.empty()) continue;
      CK(cudaEventSynchronize(p.pending.back().second));
      for (size_t i = 0; i < p.pending.size(); ++i) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, p.pending[i].first, p.pending[i].second));
        p.ms += ms;
        p.fl += p.pflops[i];
        p.en += p.pentries[i];
        p.launches += 1;
        ev_pool.push_back(p.pending[i].first);
        ev_pool.push_back(p.pending[i].second);
      }
      p.pending.clear();
      p.pflops.clear();
      p.pentries.clear();
    }
  }

  // library handles for the one-off k x k preconditioner factorisation
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solver = nullptr;
  void ensure_handles() {
    if (!blas) {
      CB(cublasCreate(&blas));
      CB(cublasSetStream(blas, st));
    }
    if (!solver) {
      CS(cusolverDnCreate(&solver));
      CS(cusolverDnSetStream(solver, st));
    }
  }
  void release_handles() {
    if (blas) cublasDestroy(blas);
    if (solver) cusolverDnDestroy(solver);
    blas = nullptr;
    solver = nullptr;
  }

  // ---- side stream: the derivative factors dL (needed only by the backward pass) are built
  // on st2 while the forward solve runs on st; every other API entry (guard) and the
  // backward pass first make st wait for that work (join_dl), and the host reads the
  // tr(P^-1 dP_w) values only when it needs them (need_trace).
  cudaStream_t st2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_dl = nullptr;
  bool dl_pending = false, trace_pending = false;
  DBuf<double> w_trace;
  bool use_side = [] {  // env GPK_SIDE_DL=0 builds dL on the main stream (A/B checks)
    const char* e = std::getenv("GPK_SIDE_DL");
    return !(e && std::atoi(e) == 0);
  }();
  void ensure_side() {
    if (!st2) CK(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
    if (!ev_fork) CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    if (!ev_dl) CK(cudaEventCreateWithFlags(&ev_dl, cudaEventDisableTiming));
  }
  void join_dl() {
    if (!dl_pending) return;
    CK(cudaStreamWaitEvent(st, ev_dl, 0));
    dl_pending = false;
  }
  void need_trace() {
    join_dl();
    if (!trace_pending) return;
    const int nw = d + 1;
    std::vector<double> hv(nw);
    CK(cudaMemcpyAsync(hv.data(), w_trace.p, sizeof(double) * nw, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int w = 0; w < nw; ++w) trace_det[w] = 2.0 * hv[w];
    trace_pending = false;
  }
  // The backward pass's preconditioner terms need only the probes, L, C and dL, so with
  // shared probes they are computed on st2 concurrently with the forward solve:
  // out[w l + i] = t_{w,i} (w <= d, precond_trace_terms_kernel), out[(d+1) l + i] = z_i' P^-1 z_i;
  // Zc receives the gathered probe block (allocated on st, read there after the join).
  cudaEvent_t ev_terms = nullptr;
  void launch_side_terms(const double* Zb, long long ldzb, int l, double* Zc, double* out) {
    ensure_side();
    if (!ev_terms) CK(cudaEventCreateWithFlags(&ev_terms, cudaEventDisableTiming));
    CK(cudaEventRecord(ev_fork, st));  // the probe block, Zc and out exist on st
    CK(cudaStreamWaitEvent(st2, ev_fork, 0));
    cudaStream_t s2 = st2;
    tl_stream = s2;
    struct Restore {
      gpk_ctx* c;
      ~Restore() { tl_stream = c->st; }
    } restore{this};
    {
      const int nw = d + 1, kw = nw * k;
      DBuf<double> Q, part, W, A, Bq, Bz, partw, dpart;
      Q.ensure(static_cast<size_t>(l) * ldn);
      part.ensure(gpk::g1_workspace(nl, k, l));
      W.ensure(static_cast<size_t>(k) * l);
      check_launch(gpk::launch_gather_cols(Zb, ldzb, nullptr, 1.0, nl, l, Zc, ldn, s2), 1, "gather");
      // Q = P^-1 Zc (psolve with its own workspaces)
      check_launch(gpk::launch_g1(L.p, n, k, Zc, ldn, l, nl, part.p, W.p, k, s2), 2, "g1");
      check_launch(gpk::launch_woodbury_apply(C.p, n, k, W.p, k, Zc, ldn, pnoise, l, nl, Q.p, ldn, s2), 1,
                   "woodbury");
      const int nrb = gpk::num_chunks(nl);
      dpart.ensure(static_cast<size_t>(l) * nrb);
      check_launch(gpk::launch_dot_partials(0, Zc, Q.p, 0.0, nl, ldn, l, dpart.p, s2), 1, "dots");
      check_launch(gpk::launch_reduce_partials(dpart.p, nrb, l, out + static_cast<size_t>(nw) * l, s2), 1, "reduce");
      A.ensure(static_cast<size_t>(2) * l * k);
      check_launch(gpk::launch_g1(L.p, n, k, Q.p, ldn, l, nl, part.p, A.p, k, s2), 2, "g1");
      check_launch(gpk::launch_g1(L.p, n, k, Zc, ldn, l, nl, part.p, A.p + static_cast<size_t>(l) * k, k, s2), 2,
                   "g1");
      Bq.ensure(static_cast<size_t>(l) * kw);
      Bz.ensure(static_cast<size_t>(l) * kw);
      partw.ensure(gpk::g1_workspace(nl, kw, l));
      check_launch(gpk::launch_g1(dL.p, n, kw, Q.p, ldn, l, nl, partw.p, Bq.p, kw, s2), 2, "g1");
      check_launch(gpk::launch_g1(dL.p, n, kw, Zc, ldn, l, nl, partw.p, Bz.p, kw, s2), 2, "g1");
      precond_trace_terms_kernel<<<static_cast<unsigned>((nw * l * 32 + 255) / 256), 256, 0, s2>>>(
          Bq.p, Bz.p, A.p, k, kw, l, nw, out);
      check_launch(cudaGetLastError(), 1, "precond_trace_terms");
    }
    CK(cudaEventRecord(ev_terms, s2));
  }
  void release_side() {
    if (ev_terms) cudaEventDestroy(ev_terms);
    ev_terms = nullptr;
    if (st2) {
      cudaStreamSynchronize(st2);
      cudaStreamDestroy(st2);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_dl) cudaEventDestroy(ev_dl);
    st2 = nullptr;
    ev_fork = ev_dl = nullptr;
  }

  void set_device() { CK(cudaSetDevice(device)); }
  void sync() { CK(cudaStreamSynchronize(st)); }
  void check_launch(cudaError_t e, int count, const char* what) {
    if (e != cudaSuccess) fail(GPK_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
    launches += count;
  }
  void h2d(void* dst, const void* src, size_t bytes) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
  }
  void d2h(void* dst, const void* src, size_t bytes) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    sync();
  }

  void require_ready() {
    require(have_data, "gpkrylov_cuda: no data set (gpk_set_data)");
    require(have_params, "gpkrylov_cuda: no hyperparameters set (gpk_set_params)");
    require(static_cast<int>(log_ls.size()) == d, "KernelOperator: lengthscale count must equal data dimension");
    if (!packed) pack();
  }

  // kernels.hpp:166-168 + packed MVM operands
  void pack() {
    X32.ensure(static_cast<size_t>(n_pad) * dp);
    X64s.ensure(static_cast<size_t>(n_pad) * dp);
    sx.ensure(static_cast<size_t>(n) * d);
    sq.ensure(n);
    ls_dev.ensure(d);
    h2d(ls_dev.p, ls.data(), sizeof(double) * d);
    check_launch(gpk::launch_pack_x(X.p, n, n, d, n_pad, ls_dev.p, gpk::prescale_c(family), dp, X32.p, dp, X64s.p,
                                    sx.p, sq.p, st),
                 1, "pack_x");
    gram_ok = false;
    tcg_direct = false;
    // Gram variant: RBF / Matern-3/2 / Matern-5/2, d <= 30, and centred pre-scaled
    // coordinates small enough that the expanded-distance cancellation stays at the
    // fp32 level (max |x~|^2 <= kGramMaxNorm; see gpk_mvm_tcg.cuh).
    if (mvm_variant != GPK_MVM_DIRECT && family != gpk::kMatern12 && d <= gpk::kGramMaxDim) {
      Xgh.ensure(static_cast<size_t>(n_pad) * 64);  // B-side then A-side augmented images
      Xgl.ensure(static_cast<size_t>(n_pad) * 64);
      Xgn.ensure(static_cast<size_t>(n_pad) + n_pad / 64);  // norms, then per-j-tile maxima
      Xgmu.ensure(d);
      check_launch(gpk::launch_gram_pack(X.p, n, n, d, n_pad, ls_dev.p, gpk::prescale_c(family), Xgmu.p, Xgh.p, Xgl.p,
                                         Xgn.p, st),
                   2, "gram_pack");
      std::vector<float> nr(n);
      d2h(nr.data(), Xgn.p, sizeof(float) * n);
      gram_maxnorm = 0.0f;
      for (float v : nr) gram_maxnorm = std::max(gram_maxnorm, v);
      gram_ok = mvm_variant == GPK_MVM_GRAM || (gram_maxnorm <= kGramMaxNorm && d >= kGramMinDim);
    }
    // low dimension (or Matern-1/2, or large norms): direct differences on the tcgen05 pipeline
    tcg_direct = !gram_ok && mvm_variant != GPK_MVM_GRAM && dp <= 8;
    packed = true;
  }
  // measured (tools/gram_check.py): C5 data with max |x~|^2 = 423 gives 1.3e-6 relative MVM error
  // with the Gram path vs 7e-7 direct -- the guard bounds the relative error in s independently
  // of the norms; the bound only excludes pathological scales
  static constexpr float kGramMaxNorm = 4096.0f;
  static constexpr int kGramMinDim = 6;  // below, direct differences cost about as much as the Gram path

  // split-K factor: a function of n only (so a column's summation order never
  // depends on t), chosen so the grid fills whole waves of 2 x 148 CTA slots
  int splits_for() const {
    const int rb = n_pad / 128;
    const int ntiles = n_pad / 32;
    const double slots = 2.0 * 148.0;
    int best = 1;
    double best_eff = 0.0;
    const int smax = std::max(1, std::min(64, ntiles / 8));
    for (int s = 1; s <= smax; ++s) {
      const int per = (ntiles + s - 1) / s;
      const int se = (ntiles + per - 1) / per;  // effective splits
      const double wv = rb * static_cast<double>(se) / slots;
      const double eff = wv / std::ceil(wv);
      if (eff > best_eff + 0.02) {
        best_eff = eff;
        best = s;
      }
      if (wv >= 1.0 && eff >= 0.97) break;
    }
    const int per = (ntiles + best - 1) / best;
    return (ntiles + per - 1) / per;
  }

  // split-K factor of the Gram tensor-core MVM (one 576-thread CTA per SM, 64-wide
  // j-tiles): minimise waves x (tiles per CTA + per-CTA start-up, ~8 tiles); a
  // function of n (and the shard's rows) only
  int splits_for_tcg() const {
    // a function of the GLOBAL n only: a shard's rows then sum their j-tiles exactly as the
    // unsharded MVM does (bitwise-equal rows across world sizes)
    const int rb = n_pad / 128;
    const int nt64 = n_pad / 64;
    int best = 1;
    double best_cost = 1e300;
    const double sms = tcg_ctas > 0 ? tcg_ctas : 148.0;
    for (int s = 1; s <= std::min(32, nt64); ++s) {
      const int per = (nt64 + s - 1) / s;
      const int se = (nt64 + per - 1) / per;
      double cost;
      if (tcg_ctas > 0) {
        // persistent grid: the busiest CTA runs ceil(U / SMs) units of `per` tiles (+ ~1 tile of
        // unpipelined drain per unit), one start-up (~8 tiles), a row change (~4) and the split
        // reduction (fp64 partials, ~0.15 tile-times per split)
        const double units = std::ceil(static_cast<double>(rb) * se / sms);
        cost = units * (per + 1.0) + 8.0 + (se > 1 ? 4.0 + 0.15 * se : 0.0);
      } else {
        const double waves = std::ceil(static_cast<double>(rb) * se / 148.0);
        cost = waves * (per + 8.0) + (se > 1 ? 0.02 * se * rb / 148.0 * per : 0.0);
      }
      if (cost < best_cost - 1e-9) {
        best_cost = cost;
        best = se;
      }
    }
    return best;
  }

  // out[:, c] = op(V[:, c]) for c < t.  which < 0: K (noise-free, scaled o^2);
  // which == 0: dK/do; 1..d: dK/dl_j; d+1: identity (noise derivative).
  // V, out: this rank's rows (nl) of t columns; the direction block is all-gathered
  // first when sharded (every rank contracts its rows against all n columns).
  void apply_kernel(const double* Vloc, long long ldvloc, int t, double* out, long long ldo, bool fp64, int which) {
    if (t <= 0) return;
    if (which == d + 1) {
      check_launch(gpk::launch_gather_cols(Vloc, ldvloc, nullptr, 1.0, nl, t, out, ldo, st), 1, "copy");
      return;
    }
    long long ldv = 0;
    const double* V = full_cols(Vloc, ldvloc, t, &ldv);
    const int mode = which >= 1 ? gpk::kModeDls : gpk::kModeValue;
    const int chunk = fp64 ? 64 : 128;
    const int splits = splits_for();
    const int ntiles = n_pad / 32;
    const int per = (ntiles + splits - 1) / splits;
    const long long ldp = (nl + 127) / 128 * 128;  // split-K partial leading dimension (local rows)
    if (!fp64 && use_tc && which < 0) {  // tcgen05 path (value mode)
      const bool tcg = gram_ok || tcg_direct;  // the gpk_mvm_tcg.cuh pipeline
      const int cmax = tcg ? 96 : 128;
      for (int c0 = 0; c0 < t; c0 += cmax) {
        const int tc = std::min(cmax, t - c0);
        gpk::MvmArgs a{};
        a.n = n;
        a.n_pad = n_pad;
        a.t = tc;
        a.scale = o2;
        a.dp = dp;
        a.row_begin = r0;
        a.row_end = r1;
        int sp = splits;
        if (tcg) {  // 64-wide j-tiles, fp16 V with per-column scales
          const int npad = gpk::tcg_npad(tc);
          w_h16hi.ensure(static_cast<size_t>(n_pad) * npad);
          w_h16lo.ensure(static_cast<size_t>(n_pad) * npad);
          w_vmax.ensure(tc);
          w_colscale.ensure(tc);
          if (vmax_ready && c0 == 0 && tc == t) {  // maxima from the fused CG p-update
            check_launch(gpk::launch_pack_v_f16_only(V, ldv, tc, n, n_pad, npad, o2, w_vmax.p, w_colscale.p,
                                                     w_h16hi.p, w_h16lo.p, st),
                         1, "pack_v_f16");
          } else {
            check_launch(gpk::launch_pack_v_f16(V + c0 * ldv, ldv, tc, n, n_pad, npad, o2, w_vmax.p, w_colscale.p,
                                                w_h16hi.p, w_h16lo.p, st),
                         2, "pack_v_f16");
          }
          const int nt64 = n_pad / 64;
          const int sg = splits_for_tcg();
          const int per64 = (nt64 + sg - 1) / sg;
          sp = (nt64 + per64 - 1) / per64;
          a.jtiles_per_split = per64;
          a.ctas = (tcg_grid_cap > 0 && tcg_ctas > 0) ? std::min(tcg_ctas, tcg_grid_cap) : tcg_ctas;
          a.flush = tc_flush;  // 64-wide tiles: 128 entries per fp32 TMEM accumulation at the default 2
          {
            // operands of one full j sweep (fp16 V hi / lo, X images or rows, norms): beyond about half
            // the 126 MB L2 the CTAs run the units strided so that they share every j-tile in time
            const double foot = static_cast<double>(n_pad) * (4.0 * npad + (gram_ok ? 260.0 : 0.0) + 4.0 * dp);
            a.unit_order = (tcg_unit_order >= 0 ? tcg_unit_order : (foot > 64e6 ? 1 : 0)) && a.ctas > 0 && sp > 1;
          }
        } else {
          const int npad = gpk::tc_npad(tc);
          w_vhi.ensure(static_cast<size_t>(n_pad) * npad);
          w_vlo.ensure(static_cast<size_t>(n_pad) * npad);
          check_launch(gpk::launch_pack_v_tc(V + c0 * ldv, ldv, tc, n, n_pad, npad, w_vhi.p, w_vlo.p, st), 1,
                       "pack_v_tc");
          a.jtiles_per_split = per;
          a.flush = tc_flush;
        }
        const int cf[] = {2, 3, 6, 9};
        const double fl = static_cast<double>(nl) * n * (2.0 * tc + 3.0 * d + cf[family]);
        auto ev = prof_begin(0);
        auto launch = [&](double* o, int nsp) {
          return tcg ? gpk::launch_fused_kmvm_tcg(family, d, gram_ok ? 0 : dp, gram_ok ? Xgh.p : X32.p,
                                                  gram_ok ? Xgl.p : X32.p, gram_ok ? Xgn.p : X32.p, X32.p, w_h16hi.p,
                                                  w_h16lo.p,
                                                      w_colscale.p, o, a, nsp, st)
                         : gpk::launch_fused_kmvm_tc(family, dp, X32.p, w_vhi.p, w_vlo.p, o, a, nsp, st);
        };
        if (sp == 1) {
          a.ldo = ldo;
          check_launch(launch(out + c0 * ldo, 1), 1, "fused_kmvm_tc");
          prof_end(0, ev, fl, static_cast<double>(nl) * n);
        } else {
          a.ldo = ldp;
          a.split_stride = static_cast<long long>(tc) * ldp;
          w_y.ensure(static_cast<size_t>(sp) * tc * ldp);
          check_launch(launch(w_y.p, sp), 1, "fused_kmvm_tc");
          prof_end(0, ev, fl, static_cast<double>(nl) * n);
          if (defer_reduce && c0 == 0 && tc == t) {
            // the caller's next kernel (cg_pap_alpha) sums the split partials itself, in the same order
            pend = {w_y.p, sp, a.split_stride, ldp};
          } else {
            check_launch(gpk::launch_reduce_splits(w_y.p, sp, a.split_stride, tc, nl, ldp, out + c0 * ldo, ldo, st),
                         1, "reduce_splits");
          }
        }
        entries += static_cast<long long>(nl) * n;
        flops += static_cast<long long>(fl);
      }
      vmax_ready = false;
      return;
    }
    if (fp64 && which < 0 && use_f64g) {  // gpk_mvm_f64g.cu: reference-order entries, DMMA products
      const int cf[] = {2, 3, 6, 9};
      for (int c0 = 0; c0 < t; c0 += 72) {
        const int tc = std::min(72, t - c0);
        const double fl = static_cast<double>(nl) * n * (2.0 * tc + 3.0 * d + cf[family]);
        auto ev = prof_begin(2);
        check_launch(gpk::launch_fused_kmvm_f64g(family, dp, X64s.p, sq.p, n, V + c0 * ldv, ldv, tc, out + c0 * ldo,
                                                 ldo, o2, r0, r1, st),
                     1, "fused_kmvm_f64g");
        prof_end(2, ev, fl, static_cast<double>(nl) * n);
        entries += static_cast<long long>(nl) * n;
        flops += static_cast<long long>(fl);
      }
      return;
    }
    for (int c0 = 0; c0 < t; c0 += chunk) {
      const int tc = std::min(chunk, t - c0);
      const gpk::MvmShape sh = gpk::mvm_shape(tc, fp64, mode);
      const void* vp;
      if (fp64) {
        w_v64.ensure(static_cast<size_t>(n_pad) * sh.vld);
        check_launch(gpk::launch_pack_v64(V + c0 * ldv, ldv, nullptr, tc, n, n_pad, sh, w_v64.p, st), 1, "pack_v64");
        vp = w_v64.p;
      } else {
        w_v32.ensure(static_cast<size_t>(n_pad) * sh.vld);
        check_launch(gpk::launch_pack_v32(V + c0 * ldv, ldv, nullptr, tc, n, n_pad, sh, w_v32.p, st), 1, "pack_v32");
        vp = w_v32.p;
      }
      gpk::MvmArgs a{};
      a.n = n;
      a.n_pad = n_pad;
      a.t = tc;
      a.jdim = which >= 1 ? which - 1 : 0;
      a.jtiles_per_split = per;
      const double c = fp64 ? 1.0 : gpk::prescale_c(family);
      if (which < 0) a.scale = o2;
      else if (which == 0) a.scale = 2.0 * o;
      else a.scale = (-2.0 * o2 / ls[which - 1]) / c;
      const void* xp = fp64 ? static_cast<const void*>(X64s.p) : static_cast<const void*>(X32.p);
      a.row_begin = r0;
      a.row_end = r1;
      const int cf[] = {2, 3, 6, 9};
      const double fl = static_cast<double>(nl) * n * (2.0 * tc + 3.0 * d + cf[family]);
      auto ev = prof_begin(0);
      if (splits == 1) {
        a.ldo = ldo;
        a.split_stride = 0;
        check_launch(gpk::launch_fused_kmvm(fp64, family, dp, mode, xp, vp, out + c0 * ldo, a, 1, st), 1,
                     "fused_kmvm");
        prof_end(0, ev, fl, static_cast<double>(nl) * n);
      } else {
        a.ldo = ldp;
        a.split_stride = static_cast<long long>(tc) * ldp;
        w_y.ensure(static_cast<size_t>(splits) * tc * ldp);
        check_launch(gpk::launch_fused_kmvm(fp64, family, dp, mode, xp, vp, w_y.p, a, splits, st), 1, "fused_kmvm");
        prof_end(0, ev, fl, static_cast<double>(nl) * n);
        check_launch(gpk::launch_reduce_splits(w_y.p, splits, a.split_stride, tc, nl, ldp, out + c0 * ldo, ldo, st),
                     1, "reduce_splits");
      }
      entries += static_cast<long long>(nl) * n;
      flops += static_cast<long long>(fl);
    }
  }

  // Z = P^{-1} R  (identity / Woodbury, preconditioners.hpp:114-118); column-major [t][ldn]
  // Woodbury on this rank's rows: W = sum_ranks L[rows]^T R[rows] (k x t), Z = (R - C[rows] W) / s2
  void psolve(const double* R, int t, double* Z) {
    if (t <= 0) return;
    if (pkind == 1) {
      check_launch(gpk::launch_gather_cols(R, ldn, nullptr, 1.0, nl, t, Z, ldn, st), 1, "copy");
      return;
    }
    if (k == 0) {
      check_launch(gpk::launch_woodbury_finish(R, nullptr, pnoise, nl, ldn, t, Z, st), 1, "woodbury");
      return;
    }
    w_g1.ensure(gpk::g1_workspace(nl, k, t));
    w_W.ensure(static_cast<size_t>(k) * t);
    w_T.ensure(static_cast<size_t>(t) * ldn);
    check_launch(gpk::launch_g1(Lloc(), ldP, k, R, ldn, t, nl, w_g1.p, w_W.p, k, st), 2, "g1");
    allreduce_sum(w_W.p, static_cast<long long>(k) * t);
    check_launch(gpk::launch_woodbury_apply(Cloc(), ldP, k, w_W.p, k, R, ldn, pnoise, t, nl, Z, ldn, st), 1,
                 "woodbury");
  }

  // per-column dots a.b over all rows (host result, fixed-order reduction, rank-ordered sum)
  std::vector<double> col_dots(const double* A, const double* B, int t, long long ld) {
    std::vector<double> out(t);
    if (t <= 0) return out;
    const int nrb = gpk::num_chunks(nl);
    w_part.ensure(static_cast<size_t>(t) * nrb * 3 + t);
    check_launch(gpk::launch_dot_partials(0, A, B, 0.0, nl, ld, t, w_part.p, st), 1, "dots");
    double* res = w_part.p + static_cast<size_t>(t) * nrb * 3;
    check_launch(gpk::launch_reduce_partials(w_part.p, nrb, t, res, st), 1, "reduce");
    allreduce_sum(res, t);
    d2h(out.data(), res, sizeof(double) * t);
    return out;
  }
  // per-slot dot partials -> (partials, nrb) consumed by the cg_* kernels: the local chunk
  // partials on one rank, else the rank-ordered global totals (nrb = 1)
  const double* global_partials(double* part, int nrb, int t, double* tot, int* nrb_out) {
    if (world == 1) {
      *nrb_out = nrb;
      return part;
    }
    check_launch(gpk::launch_reduce_partials(part, nrb, t, tot, st), 1, "reduce");
    allreduce_sum(tot, t);
    *nrb_out = 1;
    return tot;
  }

  // -------------------------------------------------------------------------
  // Batched PCG (krylov.hpp:47-129 per column, batched_pcg semantics :131-153).
  // B, Xout: device column-major with leading dimensions.  Histories are host
  // arrays [t][max_iters] (nullable).
  // -------------------------------------------------------------------------
  struct CgOut {
    std::vector<int> iters, converged, status;
    std::vector<double> bad, norm0;
    std::vector<double> pres;  // last preconditioned residual norm of the CG recurrence (krylov.hpp:102)
    // max over columns with b != 0 of pres / norm0, and the number of columns that hit max_iters
    double max_rel_pres() const {
      double m = 0.0;
      for (size_t c = 0; c < pres.size(); ++c)
        if (norm0[c] > 0.0) m = std::max(m, pres[c] / norm0[c]);
      return m;
    }
    int unconverged() const {
      int u = 0;
      for (size_t c = 0; c < converged.size(); ++c) u += converged[c] ? 0 : 1;
      return u;
    }
  };
  CgOut mbcg(const double* B, long long ldb, int t, int max_iters, double rel_tol, bool fp64, double* Xout,
             long long ldx, double* alpha_h, double* beta_h, double* resid_h,
             const std::vector<double>* tol_scale = nullptr) {
    require(max_iters >= 1, "CgConfig: max_iters must be >= 1");
    require(rel_tol > 0.0 && rel_tol < 1.0, "CgConfig: rel_tol must be in (0, 1)");
    CgOut out;
    out.iters.assign(t, 0);
    out.converged.assign(t, 0);
    out.status.assign(t, 0);
    out.bad.assign(t, 0.0);
    out.norm0.assign(t, 0.0);
    out.pres.assign(t, 0.0);
    if (t <= 0) return out;
    const int nrb = gpk::num_chunks(nl);
    for (int b = 0; b < 2; ++b) {
      st_X[b].ensure(static_cast<size_t>(t) * ldn);
      st_R[b].ensure(static_cast<size_t>(t) * ldn);
      st_P[b].ensure(static_cast<size_t>(t) * ldn);
      w_ss[b].ensure(t);
    }
    st_Z.ensure(static_cast<size_t>(t) * ldn);
    w_kx.ensure(static_cast<size_t>(t) * ldn);
    w_part.ensure(static_cast<size_t>(t) * nrb * 3 + 3 * static_cast<size_t>(t));
    w_map.ensure(t);
    const bool hist = alpha_h || beta_h || resid_h;
    if (hist) w_hist.ensure(static_cast<size_t>(3) * t * max_iters);
    double* dh_a = hist ? w_hist.p : nullptr;
    double* dh_b = hist ? w_hist.p + static_cast<size_t>(t) * max_iters : nullptr;
    double* dh_r = hist ? w_hist.p + static_cast<size_t>(2) * t * max_iters : nullptr;
    if (hist) {
      const long long cnt = 3LL * t * max_iters;
      fill_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, st>>>(w_hist.p, cnt, 0.0);
      check_launch(cudaGetLastError(), 1, "fill");
    }
    int cur = 0, compactions = 0;
    double *Xs = st_X[0].p, *Rs = st_R[0].p, *Ps = st_P[0].p, *Zs = st_Z.p;
    double* Rspare = st_R[1].p;  // r is double-buffered by pointer (the fused x/r update writes a new block)
    gpk::SlotState* ss = w_ss[0].p;
    std::vector<gpk::SlotState> hs(t);
    for (int s = 0; s < t; ++s) {
      std::memset(&hs[s], 0, sizeof(gpk::SlotState));
      hs[s].col = s;
    }
    h2d(ss, hs.data(), sizeof(gpk::SlotState) * t);
    // x0 = 0, r = b, z = P^{-1} r, norm0 = ||z||, p = z, rz = r.z   (krylov.hpp:55-67)
    check_launch(gpk::launch_gather_cols(nullptr, 0, nullptr, 0.0, nl, t, Xs, ldn, st), 1, "zero");
    check_launch(gpk::launch_gather_cols(B, ldb, nullptr, 1.0, nl, t, Rs, ldn, st), 1, "gather");
    psolve(Rs, t, Zs);
    double* prz = w_part.p;
    double* pzz = w_part.p + static_cast<size_t>(t) * nrb;
    double* ppap = w_part.p + static_cast<size_t>(2) * t * nrb;
    check_launch(gpk::launch_dot_partials(0, Rs, Zs, 0.0, nl, ldn, t, prz, st), 1, "dots");
    check_launch(gpk::launch_dot_partials(0, Zs, Zs, 0.0, nl, ldn, t, pzz, st), 1, "dots");
    double* tot = w_part.p + static_cast<size_t>(3) * t * nrb;  // global totals (sharded)
    int nrg = nrb;
    const double* grz = global_partials(prz, nrb, t, tot, &nrg);
    const double* gzz = global_partials(pzz, nrb, t, tot + t, &nrg);
    check_launch(gpk::launch_cg_init(grz, gzz, nrg, t, ss, st), 1, "cg_init");
    check_launch(gpk::launch_gather_cols(Zs, ldn, nullptr, 1.0, nl, t, Ps, ldn, st), 1, "copy");
    d2h(hs.data(), ss, sizeof(gpk::SlotState) * t);
    for (int s = 0; s < t; ++s) out.norm0[s] = hs[s].norm0;
    int ta = t;
    // per-column tolerance (defect-correction passes use absolute targets)
    auto tol_of = [&](int col) { return tol_scale ? rel_tol * (*tol_scale)[col] : rel_tol; };
    // slots whose columns differ in tolerance are handled through SlotState.norm0 scaling
    if (tol_scale) {
      for (int s = 0; s < t; ++s) hs[s].norm0 = hs[s].norm0 * tol_of(hs[s].col) / rel_tol;
      h2d(ss, hs.data(), sizeof(gpk::SlotState) * t);
    }
    auto finish_slots = [&](const std::vector<int>& done) {
      // scatter the finished columns' solutions to Xout
      if (done.empty()) return;
      std::vector<int> slots, cols;
      for (int s : done) {
        slots.push_back(s);
        cols.push_back(hs[s].col);
      }
      // gather finished slots into w_kx then scatter by column
      h2d_ring(w_map.p, slots.data(), sizeof(int) * slots.size());
      check_launch(gpk::launch_gather_cols(Xs, ldn, w_map.p, 1.0, nl, static_cast<int>(slots.size()), w_kx.p, ldn, st),
                   1, "gather");
      h2d_ring(w_map.p, cols.data(), sizeof(int) * cols.size());
      check_launch(gpk::launch_scatter_cols(w_kx.p, ldn, w_map.p, nl, static_cast<int>(cols.size()), Xout, ldx, st), 1,
                   "scatter");
      if (!use_pipe) sync();
    };
    auto compact = [&](const std::vector<int>& keep) {
      const int nt = static_cast<int>(keep.size());
      const int nb = cur ^ 1;
      if (nt > 0) {
        h2d_ring(w_map.p, keep.data(), sizeof(int) * nt);
        check_launch(gpk::launch_gather_cols(Xs, ldn, w_map.p, 1.0, nl, nt, st_X[nb].p, ldn, st), 1, "compact");
        check_launch(gpk::launch_gather_cols(Rs, ldn, w_map.p, 1.0, nl, nt, Rspare, ldn, st), 1, "compact");
        check_launch(gpk::launch_gather_cols(Ps, ldn, w_map.p, 1.0, nl, nt, st_P[nb].p, ldn, st), 1, "compact");
        // slot states gathered on the device: with the pipelined read-back the host copy is
        // one iteration old, the device copy is current
        gather_slots_kernel<<<(nt + 127) / 128, 128, 0, st>>>(ss, w_map.p, nt, w_ss[nb].p);
        check_launch(cudaGetLastError(), 1, "compact");
        std::vector<gpk::SlotState> ns(nt);
        for (int q = 0; q < nt; ++q) ns[q] = hs[keep[q]];
        if (!use_pipe) sync();
        hs = ns;
        ++compactions;
      } else {
        hs.clear();
      }
      cur = nb;
      Xs = st_X[cur].p;
      if (nt > 0) std::swap(Rs, Rspare);
      Ps = st_P[cur].p;
      vmax_ready = false;
      ss = w_ss[cur].p;
      ta = nt;
    };
    auto handle_flags = [&]() {
      std::vector<int> done, keep;
      for (int s = 0; s < ta; ++s) {
        const gpk::SlotState& x = hs[s];
        if (x.flag == gpk::kFlagError) {
          out.status[x.col] = x.status;
          out.bad[x.col] = x.bad;
          out.iters[x.col] = x.iters;
        }
      }
      // errors: report the lowest column first (reference solves y before the probes)
      int worst = -1;
      for (int s = 0; s < ta; ++s)
        if (hs[s].flag == gpk::kFlagError && (worst < 0 || hs[s].col < hs[worst].col)) worst = s;
      if (worst >= 0) {
        const gpk::SlotState& x = hs[worst];
        std::string m = "pcg_solve: breakdown at iteration " + std::to_string(x.iters);
        if (x.status == gpk::kStatusAlpha)
          m += " (alpha = " + num(x.bad) + "); operator or preconditioner not positive definite";
        else
          m += " (r'z = " + num(x.bad) + ")";
        throw GpkError{GPK_SOLVER_ERROR, "#col" + std::to_string(x.col) + "#" + m};
      }
      for (int s = 0; s < ta; ++s) {
        if (hs[s].flag == gpk::kFlagConverged) {
          out.iters[hs[s].col] = hs[s].iters;
          out.pres[hs[s].col] = hs[s].pres;
          out.converged[hs[s].col] = 1;
          done.push_back(s);
        } else {
          keep.push_back(s);
        }
      }
      if (!done.empty()) {
        finish_slots(done);
        compact(keep);
      }
    };
    handle_flags();  // zero right-hand sides finish with 0 iterations
    // single-rank Woodbury path: the fused iteration (gpk_cgfused.cu)
    const bool fused = use_fused_cg && world == 1 && pkind == 2 && k > 0;
    if (fused) {
      w_cnt.ensure(static_cast<size_t>(t) + 64);
      CK(cudaMemsetAsync(w_cnt.p, 0, sizeof(unsigned) * (static_cast<size_t>(t) + 64), st));
      const int nbx = gpk::g2_row_blocks(nl);
      w_prz.ensure(static_cast<size_t>(t) * nbx);
      w_pzz.ensure(static_cast<size_t>(t) * nbx);
      w_g1.ensure(gpk::g1_workspace(nl, k, t));
      w_W.ensure(static_cast<size_t>(k) * t);
      w_vmax.ensure(t);
      if (use_wood_s) {
        w_g1.ensure(gpk::wood_g1_workspace(k, t));
        w_prz.ensure(gpk::wood_g2_partials(t));
        w_pzz.ensure(gpk::wood_g2_partials(t));
        w_cnt2.ensure(t);
        CK(cudaMemsetAsync(w_cnt2.p, 0, sizeof(unsigned) * t, st));
        if (use_coop) w_ppap.ensure(gpk::wood_g2_partials(t));
      }
    }
    // pipelined read-back: snapshot of iteration it (async), then the decision on the
    // snapshot of iteration it - 1 (already complete while iteration it runs).  A snapshot
    // taken before a compaction has the old slot layout and is skipped.
    int pend_buf = -1;
    snap_h.ensure(sizeof(gpk::SlotState) * 2 * static_cast<size_t>(t));
    auto* snaps = reinterpret_cast<gpk::SlotState*>(snap_h.p);
    // written_by_kernel: the iteration's last kernel already stored the snapshot into the
    // pinned buffer (no copy-engine round trip)
    auto readback = [&](int it, bool written_by_kernel = false) {
      const int bcur = it & 1;
      if (!written_by_kernel)
        CK(cudaMemcpyAsync(snaps + static_cast<size_t>(bcur) * t, ss, sizeof(gpk::SlotState) * ta,
                           cudaMemcpyDeviceToHost, st));
      CK(cudaEventRecord(snap_ev.get(bcur), st));
      const int take = it == max_iters ? bcur : pend_buf;  // the last iteration drains
      pend_buf = bcur;
      if (take < 0) return;
      CK(cudaEventSynchronize(snap_ev.get(take)));
      std::memcpy(hs.data(), snaps + static_cast<size_t>(take) * t, sizeof(gpk::SlotState) * ta);
      const int c0 = compactions;
      handle_flags();
      if (compactions != c0) pend_buf = -1;  // the in-flight snapshot has the old layout
    };
    vmax_ready = false;
    for (int it = 1; it <= max_iters && ta > 0; ++it) {
      w_kx.ensure(static_cast<size_t>(ta) * ldn);
      // fused iteration on one rank: the split-K partials of K p are summed by the p'Ap kernel
      pend = PendingSplits{};
      defer_reduce = fused && fuse_reduce && world == 1 && !(use_wood_s && use_coop);
      apply_kernel(Ps, ldn, ta, w_kx.p, ldn, fp64, -1);  // K p (noise-free)
      defer_reduce = false;
      if (fused) {
        // vector phase (kind 3): algorithmic HBM bytes = 13 fp64 n-vectors per column (pap: P, Kp;
        // x/r update: R, P, Kp, X read, X, R written; Woodbury: R read, Z written; p update: P, Z
        // read, P written) + L and C (n x k fp64 each)
        auto evv = prof_begin(3);
        const double vbytes = 8.0 * nl * (13.0 * ta + 2.0 * k);
        unsigned long long* vm = (!fp64 && use_tc && (gram_ok || tcg_direct) && ta <= 96) ? w_vmax.p : nullptr;
        if (!(use_wood_s && use_coop))
          check_launch(gpk::launch_cg_pap_alpha(Ps, w_kx.p, noise, nl, ldn, ta, ppap, w_cnt.p, it, ss, dh_a,
                                                max_iters, st, use_wood_s ? vm : nullptr, pend.part, pend.splits,
                                                pend.sstride, pend.ldp),
                       1, "cg_pap_alpha");
        if (use_wood_s && use_coop) {  // gpk_wood.cu: the whole vector phase in one cooperative launch
          check_launch(gpk::launch_cg_iter_coop(L.p, n, C.p, n, k, Xs, Rs, Ps, Zs, w_kx.p, ldn, ta, nl, noise, pnoise,
                                                w_ppap.p, w_g1.p, w_W.p, w_prz.p, w_pzz.p, ss, it, rel_tol, dh_a, dh_b,
                                                dh_r, max_iters, vm,
                                                use_pipe ? snaps + static_cast<size_t>(it & 1) * t : nullptr, st),
                       1, "cg_iter_coop");
        } else if (use_wood_s) {  // gpk_wood.cu: x/r update fused into the staged G1, staged G2 + dots, beta + p
          check_launch(gpk::launch_g1s(L.p, n, k, Rs, ldn, ta, nl, w_g1.p, w_W.p, k, Xs, Ps, w_kx.p, noise, ss, st),
                       2, "g1s");
          check_launch(gpk::launch_g2s_dots_beta(C.p, n, k, w_W.p, k, ta, nl, Zs, Rs, ldn, pnoise, w_prz.p, w_pzz.p,
                                                 st),
                       (ta + 63) / 64, "g2s_dots");
          check_launch(gpk::launch_cg_beta_p(Ps, Zs, nl, ldn, ta, ss, w_prz.p, w_pzz.p, w_cnt2.p, it, rel_tol, dh_b,
                                             dh_r, max_iters, vm,
                                             use_pipe ? snaps + static_cast<size_t>(it & 1) * t : nullptr, st),
                       1, "cg_beta_p");
        } else {
          check_launch(gpk::launch_cg_update_xr(Xs, Rs, Ps, w_kx.p, noise, nl, ldn, ta, ss, st), 1, "cg_xr");
          check_launch(gpk::launch_g1(L.p, n, k, Rs, ldn, ta, nl, w_g1.p, w_W.p, k, st), 2, "g1");
          check_launch(gpk::launch_g2_dots_beta(C.p, n, k, w_W.p, k, ta, nl, Zs, Rs, ldn, pnoise, w_prz.p, w_pzz.p,
                                                w_cnt.p + t, it, rel_tol, ss, dh_b, dh_r, max_iters, vm, st),
                       1, "g2_dots_beta");
          check_launch(gpk::launch_cg_p_vmax(Ps, Zs, nl, ldn, ta, ss, vm, st), 1, "cg_p");
        }
        prof_end(3, evv, vbytes, static_cast<double>(ta));
        vmax_ready = vm != nullptr;
        if (use_pipe) {
          readback(it, use_wood_s);
          continue;
        }
        if (it % sync_every == 0 || it == max_iters) {
          d2h(hs.data(), ss, sizeof(gpk::SlotState) * ta);
          handle_flags();
        }
        continue;
      }
      check_launch(gpk::launch_dot_partials(1, Ps, w_kx.p, noise, nl, ldn, ta, ppap, st), 1, "dots");
      const double* gpap = global_partials(ppap, nrb, ta, tot + 2 * t, &nrg);
      check_launch(gpk::launch_cg_alpha(gpap, nrg, ta, it, ss, dh_a, max_iters, st), 1, "cg_alpha");
      check_launch(gpk::launch_cg_update_xr(Xs, Rs, Ps, w_kx.p, noise, nl, ldn, ta, ss, st), 1, "cg_xr");
      psolve(Rs, ta, Zs);
      check_launch(gpk::launch_dot_partials(0, Rs, Zs, 0.0, nl, ldn, ta, prz, st), 1, "dots");
      check_launch(gpk::launch_dot_partials(0, Zs, Zs, 0.0, nl, ldn, ta, pzz, st), 1, "dots");
      const double* grz2 = global_partials(prz, nrb, ta, tot, &nrg);
      const double* gzz2 = global_partials(pzz, nrb, ta, tot + t, &nrg);
      check_launch(gpk::launch_cg_beta(grz2, gzz2, nrg, ta, it, rel_tol, ss, dh_b, dh_r, max_iters, st), 1, "cg_beta");
      check_launch(gpk::launch_cg_update_p(Ps, Zs, nl, ldn, ta, ss, st), 1, "cg_p");
      if (use_pipe) {
        readback(it);
        continue;
      }
      // Host round trip only every sync_every iterations: converged / failed columns freeze
      // on the device (their flag) and are compacted out at the next sync.
      if (it % sync_every == 0 || it == max_iters) {
        d2h(hs.data(), ss, sizeof(gpk::SlotState) * ta);
        handle_flags();
      }
    }
    vmax_ready = false;
    // columns that hit max_iters: not an error, converged = false (krylov.hpp:120)
    if (ta > 0) {
      std::vector<int> all;
      for (int s = 0; s < ta; ++s) {
        out.iters[hs[s].col] = hs[s].iters;
        out.pres[hs[s].col] = hs[s].pres;
        all.push_back(s);
      }
      finish_slots(all);
    }
    if (hist) {
      std::vector<double> h(static_cast<size_t>(3) * t * max_iters);
      d2h(h.data(), w_hist.p, sizeof(double) * h.size());
      const size_t blk = static_cast<size_t>(t) * max_iters;
      if (alpha_h) std::memcpy(alpha_h, h.data(), sizeof(double) * blk);
      if (beta_h) std::memcpy(beta_h, h.data() + blk, sizeof(double) * blk);
      if (resid_h) std::memcpy(resid_h, h.data() + 2 * blk, sizeof(double) * blk);
    }
    return out;
  }

  // FP32 defect correction: audit the fp64 preconditioned true residual of
  // every column and correct the converged ones above tolerance.  The fp64
  // residual R = B - K_hat X is formed ONCE (fp64 fused MVM); after a correction
  // X += E it is updated as R -= K_hat E with the solve's own (reduced-precision)
  // operator: E is the small defect, so that product's relative error (<= ~5e-7)
  // perturbs R by ~5e-7 |R|, far below the tolerance being certified.
  // *max_ratio = max over all columns with b != 0 (converged or not: a column that hit
  // max_iters shows its true residual); -1 when no column converged — nothing can be
  // certified then, and the fp64 residual MVM is skipped (the CG recurrence's own residual
  // is reported by the caller instead, CgOut::max_rel_pres).
  int refine(const double* B, long long ldb, int t, double* Xd, long long ldx, const CgOut& cg, int max_iters,
             double rel_tol, int passes, double* max_ratio) {
    int nconv = 0;
    for (int c = 0; c < t; ++c) nconv += (cg.converged[c] && cg.norm0[c] > 0.0) ? 1 : 0;
    *max_ratio = -1.0;
    if (nconv == 0) return 0;
    w_tmp.ensure(static_cast<size_t>(t) * ldn);
    w_tmp2.ensure(static_cast<size_t>(t) * ldn);
    w_B.ensure(static_cast<size_t>(t) * ldn);
    int used = 0;
    // R = B - (K X + s2 X)  in fp64
    w_kx.ensure(static_cast<size_t>(t) * ldn);
    apply_kernel(Xd, ldx, t, w_kx.p, ldn, true, -1);
    check_launch(gpk::launch_gather_cols(Xd, ldx, nullptr, 1.0, nl, t, w_tmp2.p, ldn, st), 1, "copy");
    {
      dim3 g((nl + 255) / 256, t);
      residual_kernel<<<g, 256, 0, st>>>(B, ldb, w_kx.p, w_tmp2.p, noise, nl, ldn, w_B.p);
      check_launch(cudaGetLastError(), 1, "residual");
    }
    for (int pass = 0; pass <= passes; ++pass) {
      psolve(w_B.p, t, w_tmp.p);
      const std::vector<double> zz = col_dots(w_tmp.p, w_tmp.p, t, ldn);
      std::vector<int> bad;
      std::vector<double> scale;
      double mr = 0.0;
      for (int c = 0; c < t; ++c) {
        if (cg.norm0[c] == 0.0) continue;
        const double ratio = std::sqrt(zz[c]) / cg.norm0[c];
        mr = std::max(mr, ratio);
        if (ratio > rel_tol && cg.converged[c]) {  // a capped column cannot be certified by correction
          bad.push_back(c);
          scale.push_back(cg.norm0[c] / std::sqrt(zz[c]));
        }
      }
      *max_ratio = mr;
      if (std::getenv("GPK_DEBUG_REFINE"))
        std::fprintf(stderr, "[refine] pass %d: t=%d bad=%zu max_ratio=%.3e\n", pass, t, bad.size(), mr);
      if (bad.empty() || pass == passes) break;
      ++used;
      // correction solve K E = R[:, bad] with absolute target rel_tol * norm0
      const int nb = static_cast<int>(bad.size());
      DBuf<double> Rb, Eb, KE;
      Rb.ensure(static_cast<size_t>(nb) * ldn);
      Eb.ensure(static_cast<size_t>(nb) * ldn);
      KE.ensure(static_cast<size_t>(nb) * ldn);
      w_map.ensure(nb);
      h2d(w_map.p, bad.data(), sizeof(int) * nb);
      check_launch(gpk::launch_gather_cols(w_B.p, ldn, w_map.p, 1.0, nl, nb, Rb.p, ldn, st), 1, "gather");
      // relative tolerance of the correction solve: 0.5 * rel_tol * norm0 / ||P^-1 r_true|| (< 0.5)
      std::vector<double> ts(nb);
      for (int q = 0; q < nb; ++q) ts[q] = 0.5 * scale[q];
      CgOut c2 = mbcg(Rb.p, ldn, nb, max_iters, rel_tol, false, Eb.p, ldn, nullptr, nullptr, nullptr, &ts);
      (void)c2;
      // X[:, bad] += E   (the inner solve reused w_map: upload the column list again)
      h2d(w_map.p, bad.data(), sizeof(int) * nb);
      w_tmp2.ensure(static_cast<size_t>(nb) * ldn);
      check_launch(gpk::launch_gather_cols(Xd, ldx, w_map.p, 1.0, nl, nb, w_tmp2.p, ldn, st), 1, "gather");
      check_launch(gpk::launch_axpby(w_tmp2.p, Eb.p, 1.0, 1.0, nl, nb, ldn, st), 1, "axpy");
      check_launch(gpk::launch_scatter_cols(w_tmp2.p, ldn, w_map.p, nl, nb, Xd, ldx, st), 1, "scatter");
      // R[:, bad] -= K E + s2 E  (reduced-precision product of the small correction)
      apply_kernel(Eb.p, ldn, nb, KE.p, ldn, false, -1);
      {
        dim3 g((nl + 255) / 256, nb);
        residual_kernel<<<g, 256, 0, st>>>(Rb.p, ldn, KE.p, Eb.p, noise, nl, ldn, w_tmp2.p);
        check_launch(cudaGetLastError(), 1, "residual");
      }
      check_launch(gpk::launch_scatter_cols(w_tmp2.p, ldn, w_map.p, nl, nb, w_B.p, ldn, st), 1, "scatter");
      sync();
    }
    return used;
  }
};

namespace {

gpk_status guard(gpk_ctx* ctx, const std::function<void()>& f, bool defer_dl = false) {
  try {
    if (ctx) {
      ctx->set_device();
      tl_stream = ctx->st;
      if (!defer_dl) ctx->join_dl();  // side-stream derivative factors complete before any other use
    }
    f();
    if (ctx) ctx->err.clear();
    return GPK_OK;
  } catch (const GpkError& e) {
    if (ctx) ctx->err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    return GPK_NUMERICAL_ERROR;
  }
}

// Strip the internal "#colN#" prefix of an mBCG breakdown message.
std::string strip_col(const std::string& m, int* col) {
  *col = -1;
  if (m.size() > 4 && m.compare(0, 4, "#col") == 0) {
    const size_t e = m.find('#', 4);
    *col = std::stoi(m.substr(4, e - 4));
    return m.substr(e + 1);
  }
  return m;
}

uint64_t mix_seed_impl(uint64_t seed, uint64_t salt) {  // common.hpp:93-98
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void make_probes_impl(int64_t n, int count, uint64_t seed, double* out) {  // trace_estimation.hpp:27-36
  require(n >= 1, "make_probes: n must be >= 1");
  require(count >= 1, "make_probes: need at least one probe");
  std::mt19937_64 rng(seed);
  const double inv = 1.0 / std::sqrt(static_cast<double>(n));
  for (int c = 0; c < count; ++c)
    for (int64_t i = 0; i < n; ++i) out[c * n + i] = (rng() & 1ULL) ? inv : -inv;
}

// ---------------------------------------------------------------------------
// evaluate_mll (gp_likelihood.hpp:51-103) on device-resident y (n) and Z (n x l)
// ---------------------------------------------------------------------------
void evaluate_impl(gpk_ctx* c, const double* dy, const double* dZ, int64_t ldz, int l, uint64_t seed,
                   const gpk_mll_cfg* cfg, gpk_mll_result* res) {
  c->require_ready();
  require(cfg != nullptr && res != nullptr, "evaluate_mll: null config or result");
  require(l >= 1, "make_probes: need at least one probe");
  require(c->pkind != 0, "evaluate_mll: no preconditioner (gpk_pivoted_cholesky or gpk_precond_identity)");
  const int n = c->n, d = c->d, np = d + 2;
  const long long ldn = c->ldn;
  require(cfg->solver.precision >= GPK_PREC_FP64 && cfg->solver.precision <= GPK_PREC_TF32X3,
          "CgConfig: unknown precision");
  const bool fp64 = cfg->solver.precision == GPK_PREC_FP64;
  c->use_tc = cfg->solver.precision == GPK_PREC_TF32X3;
  const int mi = cfg->solver.max_iters;
  const double tol = cfg->solver.rel_tol;
  require(mi >= 1, "CgConfig: max_iters must be >= 1");
  require(tol > 0.0 && tol < 1.0, "CgConfig: rel_tol must be in (0, 1)");
  const long long launches0 = c->launches;
  c->entries = 0;
  c->flops = 0;
  struct Events {  // destroyed on every exit path (the solver errors above are recoverable)
    cudaEvent_t e[3] = {nullptr, nullptr, nullptr};
    ~Events() {
      for (cudaEvent_t& x : e)
        if (x) cudaEventDestroy(x);
    }
  } ev;
  CK(cudaEventCreate(&ev.e[0]));
  CK(cudaEventCreate(&ev.e[1]));
  CK(cudaEventCreate(&ev.e[2]));
  cudaEvent_t e0 = ev.e[0], e1 = ev.e[1], e2 = ev.e[2];
  CK(cudaEventRecord(e0, c->st));
  // unshared backward batch (gp_likelihood.hpp:79-84): its host mt19937_64 stream is drawn on a
  // host thread while the device runs the forward solve
  std::vector<double> hz_bwd;
  std::thread bwd_draw;
  if (cfg->with_gradient && !cfg->share_probes) {
    hz_bwd.resize(static_cast<size_t>(n) * l);
    bwd_draw = std::thread([&hz_bwd, n, l, seed] { make_probes_impl(n, l, mix_seed_impl(seed, 0xb2dULL), hz_bwd.data()); });
  }
  struct DrawJoin {
    std::thread& t;
    ~DrawJoin() {
      if (t.joinable()) t.join();
    }
  } draw_join{bwd_draw};

  // ---- forward: one mBCG over [y, z_1..z_l] (pcg_solve(y) + vr_logdet's probe solves)
  const int t = 1 + l;
  DBuf<double> B, Xs;
  B.ensure(static_cast<size_t>(t) * ldn);
  Xs.ensure(static_cast<size_t>(t) * ldn);
  const int nl = c->nl, r0 = c->r0;  // this rank's rows of y, Z and the CG state
  c->check_launch(gpk::launch_gather_cols(dy + r0, n, nullptr, 1.0, nl, 1, B.p, ldn, c->st), 1, "gather");
  c->check_launch(gpk::launch_gather_cols(dZ + r0, ldz, nullptr, 1.0, nl, l, B.p + ldn, ldn, c->st), 1, "gather");
  // backward preconditioner terms on the side stream, overlapped with the forward solve
  DBuf<double> Zc, dterms;  // allocated on st: read there after the join
  require(cfg->backward_mode >= 0 && cfg->backward_mode <= 3, "MllConfig: unknown backward mode");
  const bool side_terms = cfg->with_gradient && cfg->share_probes && cfg->backward_mode != 1 && c->use_side &&
                          c->pkind == 2 && c->k > 0 && c->world == 1 && c->have_dl;
  if (cfg->with_gradient) Zc.ensure(static_cast<size_t>(l) * ldn);
  if (side_terms) {
    dterms.ensure(static_cast<size_t>(d + 2) * l);
    c->launch_side_terms(dZ + r0, ldz, l, Zc.p, dterms.p);
  }
  std::vector<double> ah(static_cast<size_t>(t) * mi), bh(static_cast<size_t>(t) * mi);
  gpk_ctx::CgOut cg;
  try {
    cg = c->mbcg(B.p, ldn, t, mi, tol, fp64, Xs.p, ldn, ah.data(), bh.data(), nullptr);
  } catch (const GpkError& e) {
    if (e.code != GPK_SOLVER_ERROR) throw;
    int col;
    const std::string m = strip_col(e.msg, &col);
    if (col <= 0) fail(GPK_SOLVER_ERROR, m);  // the y solve (gp_likelihood.hpp:61)
    fail(GPK_NUMERICAL_ERROR, "vr_logdet: probe " + std::to_string(col - 1) + ": " + m);  // :177-179
  }
  res->refine_passes = 0;
  res->max_true_rel_residual = -1.0;
  res->max_cg_rel_residual = cg.max_rel_pres();
  res->unconverged_columns = cg.unconverged();
  res->backward_mode_used = cfg->backward_mode == 1 ? 1 : 0;
  if (!fp64 && cfg->solver.refine > 0) {
    double mr = -1.0;
    try {  // a breakdown inside a correction solve maps like the solve it corrects
      res->refine_passes = c->refine(B.p, ldn, t, Xs.p, ldn, cg, mi, tol, cfg->solver.refine, &mr);
    } catch (const GpkError& e) {
      if (e.code != GPK_SOLVER_ERROR) throw;
      int col;
      const std::string m = strip_col(e.msg, &col);
      if (col <= 0) fail(GPK_SOLVER_ERROR, m);
      fail(GPK_NUMERICAL_ERROR, "vr_logdet: probe " + std::to_string(col - 1) + ": " + m);
    }
    res->max_true_rel_residual = mr;
  }
  const double* U = Xs.p;
  const double* S = Xs.p + ldn;

  // ---- SLQ per probe (trace_estimation.hpp:163-176) on the host: the l tridiagonal
  // eigen-solves run on host threads while the device works on the backward pass; the
  // value is finished after the join (same per-probe arithmetic, fixed-order sums).
  std::vector<double> gam(l);
  std::vector<std::string> slq_err(l);
  auto slq_probe = [&](int i) {
    const int col = 1 + i;
    const int m = cg.iters[col];
    std::vector<double> dg, sb;
    dg.reserve(m);
    sb.reserve(m);
    for (int kk = 1; kk <= m; ++kk) {  // krylov.hpp:85-92
      const double a = ah[static_cast<size_t>(col) * mi + kk - 1];
      double dv = 1.0 / a;
      if (kk > 1) {
        const double ap = ah[static_cast<size_t>(col) * mi + kk - 2];
        const double bp = bh[static_cast<size_t>(col) * mi + kk - 2];
        dv += bp / ap;
        sb.push_back(std::sqrt(bp) / ap);
      }
      dg.push_back(dv);
    }
    try {
      gam[i] = slq_log(dg, sb).value;
    } catch (const GpkError& e) {
      slq_err[i] = e.msg;
    }
  };
  std::vector<std::thread> slq_threads;
  {
    // one launcher thread spawns the workers (creating 16 threads here stalled the stream's
    // next launch by ~0.35 ms)
    const int nth = std::max(1, std::min<int>(l, std::min(16u, std::max(1u, std::thread::hardware_concurrency()))));
    slq_threads.emplace_back([&slq_probe, l, nth] {
      std::vector<std::thread> workers;
      for (int th = 1; th < nth; ++th)
        workers.emplace_back([&slq_probe, l, nth, th] {
          for (int i = th; i < l; i += nth) slq_probe(i);
        });
      for (int i = 0; i < l; i += nth) slq_probe(i);
      for (auto& wk : workers) wk.join();
    });
  }
  auto finish_forward = [&]() {
    for (auto& th : slq_threads) th.join();
    slq_threads.clear();
    for (int i = 0; i < l; ++i) {
      if (!slq_err[i].empty()) fail(GPK_NUMERICAL_ERROR, "vr_logdet: probe " + std::to_string(i) + ": " + slq_err[i]);
      if (res->forward_cg_iterations) res->forward_cg_iterations[i] = cg.iters[1 + i];
      if (res->forward_gammas) res->forward_gammas[i] = gam[i];
    }
    const double plogdet = c->pkind == 1 ? 0.0 : c->plogdet;
    double stoch = 0.0;  // finish_estimate (trace_estimation.hpp:132-141)
    for (double g : gam) stoch += g;
    stoch *= static_cast<double>(n) / static_cast<double>(l);
    std::vector<double> scaled(l);
    for (int i = 0; i < l; ++i) scaled[i] = static_cast<double>(n) * gam[i];
    res->value_sample_variance = unbiased_variance(scaled);
    res->logdet = plogdet + stoch;
    res->logdet_precond = plogdet;
    const double kPi = 3.14159265358979323846;
    res->value = -0.5 * (res->quad + res->logdet + static_cast<double>(n) * std::log(2.0 * kPi));
  };
  struct JoinGuard {  // never leave the SLQ threads running on an error path
    std::vector<std::thread>& t;
    ~JoinGuard() {
      for (auto& th : t)
        if (th.joinable()) th.join();
    }
  } slq_guard{slq_threads};
  const double quad = c->col_dots(dy + r0, U, 1, ldn)[0];  // y.u
  res->quad = quad;
  res->solve_iterations = cg.iters[0];
  res->total_cg_iterations = 0;
  for (int col = 0; col < t; ++col) res->total_cg_iterations += cg.iters[col];
  CK(cudaEventRecord(e1, c->st));

  if (cfg->with_gradient) {
    require(res->gradient != nullptr, "evaluate_mll: null gradient buffer");
    c->need_trace();  // the side-stream derivative factors (gpk_precond_deriv_factors) are done
    // backward probe batch (gp_likelihood.hpp:79-84)
    const double* Zb = dZ + r0;  // this rank's rows of the backward batch
    long long ldzb = ldz;
    DBuf<double> Zu, Su;
    const double* Sb = S;
    long long ldsb = ldn;
    if (!cfg->share_probes) {
      bwd_draw.join();
      Zu.ensure(static_cast<size_t>(l) * ldn);
      CK(cudaMemcpy2DAsync(Zu.p, ldn * sizeof(double), hz_bwd.data() + r0, n * sizeof(double), nl * sizeof(double),
                           l, cudaMemcpyHostToDevice, c->st));
      Zb = Zu.p;
      ldzb = ldn;
    }
    // ---- preconditioner terms: Q = P^{-1} Zb, t_{w,i} = z_i' P^{-1} dP_w z_i
    DBuf<double> Q;
    std::vector<std::vector<double>> tw(np, std::vector<double>(l, 0.0));
    std::vector<double> tdet(np, 0.0);
    const bool dplr = c->pkind == 2;
    if (side_terms) {  // computed on st2 during the forward solve
      CK(cudaStreamWaitEvent(c->st, c->ev_terms, 0));
      std::vector<double> h(static_cast<size_t>(d + 2) * l);
      c->d2h(h.data(), dterms.p, sizeof(double) * h.size());
      for (int w = 0; w <= d + 1; ++w) {
        tdet[w] = c->trace_det[w];
        for (int i = 0; i < l; ++i) tw[w][i] = h[static_cast<size_t>(w) * l + i];
      }
    } else {
      Q.ensure(static_cast<size_t>(l) * ldn);
      c->check_launch(gpk::launch_gather_cols(Zb, ldzb, nullptr, 1.0, nl, l, Zc.p, ldn, c->st), 1, "gather");
      c->psolve(Zc.p, l, Q.p);
    }
    if (dplr && !side_terms) {
      tdet[d + 1] = c->trace_det[d + 1];
      const std::vector<double> zq = c->col_dots(Zc.p, Q.p, l, ldn);
      for (int i = 0; i < l; ++i) tw[d + 1][i] = zq[i];  // dP/dsigma^2 = I
      if (c->k > 0) {
        require(c->have_dl, "DiagPlusLowRank: derivative factors not attached");
        const int k = c->k;
        // [Q Zc] is contiguous: columns 0..l-1 of Q then Zc (separate buffers -> two G1s)
        DBuf<double> A, part;
        A.ensure(static_cast<size_t>(2) * l * k);
        part.ensure(gpk::g1_workspace(nl, k, l));
        c->check_launch(gpk::launch_g1(c->Lloc(), c->ldP, k, Q.p, ldn, l, nl, part.p, A.p, k, c->st), 2, "g1");
        c->check_launch(gpk::launch_g1(c->Lloc(), c->ldP, k, Zc.p, ldn, l, nl, part.p, A.p + static_cast<size_t>(l) * k,
                                       k, c->st),
                        2, "g1");
        c->allreduce_sum(A.p, 2LL * l * k);
        // all d+1 derivative factors at once: dL is [w][n x k], i.e. one n x (d+1)k matrix
        const int kw = (d + 1) * k;
        DBuf<double> Bq, Bz, partw, dtw;
        Bq.ensure(static_cast<size_t>(l) * kw);
        Bz.ensure(static_cast<size_t>(l) * kw);
        partw.ensure(gpk::g1_workspace(nl, kw, l));
        c->check_launch(gpk::launch_g1(c->dLloc(), c->ldP, kw, Q.p, ldn, l, nl, partw.p, Bq.p, kw, c->st), 2, "g1");
        c->check_launch(gpk::launch_g1(c->dLloc(), c->ldP, kw, Zc.p, ldn, l, nl, partw.p, Bz.p, kw, c->st), 2, "g1");
        c->allreduce_sum(Bq.p, static_cast<long long>(l) * kw);
        c->allreduce_sum(Bz.p, static_cast<long long>(l) * kw);
        dtw.ensure(static_cast<size_t>(d + 1) * l);
        precond_trace_terms_kernel<<<static_cast<unsigned>(((d + 1) * l * 32 + 255) / 256), 256, 0, c->st>>>(
            Bq.p, Bz.p, A.p, k, kw, l, d + 1, dtw.p);
        c->check_launch(cudaGetLastError(), 1, "precond_trace_terms");
        std::vector<double> htw(static_cast<size_t>(d + 1) * l);
        c->d2h(htw.data(), dtw.p, sizeof(double) * htw.size());
        for (int w = 0; w <= d; ++w) {
          tdet[w] = c->trace_det[w];
          for (int i = 0; i < l; ++i) tw[w][i] = htw[static_cast<size_t>(w) * l + i];
        }
      }
    }
    // ---- K_hat terms: quad_w = u' dK_w u and z_i' K_hat^{-1} dK_w z_i
    std::vector<double> quadw(np, 0.0);
    std::vector<std::vector<double>> zw(np, std::vector<double>(l, 0.0));  // z_i' w_i
    std::vector<bool> per_probe(np, true);
    // unshared batch needs its own solves s_i = K_hat^{-1} zb_i
    DBuf<double> Sx;
    if (!cfg->share_probes) {
      Sx.ensure(static_cast<size_t>(l) * ldn);
      gpk_ctx::CgOut cgb;
      try {
        cgb = c->mbcg(Zc.p, ldn, l, mi, tol, fp64, Sx.p, ldn, nullptr, nullptr, nullptr);
      } catch (const GpkError& e) {
        int col;
        const std::string m = strip_col(e.msg, &col);
        fail(GPK_NUMERICAL_ERROR, "trace residual: probe " + std::to_string(std::max(col, 0)) + ": " + m);
      }
      for (int i = 0; i < l; ++i) res->total_cg_iterations += cgb.iters[i];
      res->max_cg_rel_residual = std::max(res->max_cg_rel_residual, cgb.max_rel_pres());
      res->unconverged_columns += cgb.unconverged();
      if (!fp64 && cfg->solver.refine > 0) {
        double mr = -1.0;
        try {
          c->refine(Zc.p, ldn, l, Sx.p, ldn, cgb, mi, tol, cfg->solver.refine, &mr);
        } catch (const GpkError& e) {
          int col;
          const std::string m = strip_col(e.msg, &col);
          fail(GPK_NUMERICAL_ERROR, "trace residual: probe " + std::to_string(std::max(col, 0)) + ": " + m);
        }
        res->max_true_rel_residual = std::max(res->max_true_rel_residual, mr);
      }
      Sb = Sx.p;
      ldsb = ldn;
    }
    // noise: w_i = s_i (cached forward solves when shared, gp_likelihood.hpp:90)
    {
      const double uu = c->col_dots(U, U, 1, ldn)[0];
      quadw[d + 1] = uu;
      const std::vector<double> zs = c->col_dots(Zc.p, Sb, l, ldn);
      for (int i = 0; i < l; ++i) zw[d + 1][i] = zs[i];
    }
    // auto (2): the fused identity z' K^-1 dK z = s' dK z holds for converged solves; when a
    // forward column hit max_iters the reference's truncated estimator (per-RHS solves) is
    // reproduced instead (C1 as configured: the fused gradient's truncation error is ~3x the
    // faithful one, profiles/r2_c1_fused_truncation.txt)
    const bool fused_bwd =
        cfg->backward_mode == 0 || cfg->backward_mode == 3 || (cfg->backward_mode == 2 && cg.unconverged() == 0);
    res->backward_mode_used = fused_bwd ? 0 : 1;
    if (fused_bwd) {
      // fused bilinear derivative pass over all n^2 pairs
      const int n_pad = c->n_pad;
      const size_t elem = fp64 ? 8 : 4;
      DBuf<unsigned char> ops;
      ops.ensure(elem * static_cast<size_t>(n_pad) * (1 + 2 * l));
      unsigned char* Up = ops.p;
      unsigned char* SZp = ops.p + elem * n_pad;
      auto conv = [&](const double* src, long long lds, int tt, unsigned char* dst) {
        const long long tot = static_cast<long long>(tt) * n_pad;
        if (fp64)
          to_padded_kernel<double><<<static_cast<unsigned>((tot + 255) / 256), 256, 0, c->st>>>(
              src, lds, n, n_pad, tt, reinterpret_cast<double*>(dst));
        else
          to_padded_kernel<float><<<static_cast<unsigned>((tot + 255) / 256), 256, 0, c->st>>>(
              src, lds, n, n_pad, tt, reinterpret_cast<float*>(dst));
        c->check_launch(cudaGetLastError(), 1, "to_padded");
      };
      // the b-side of the pairs runs over all n rows: all-gather u, S, Z when sharded
      const double *Uall = U, *Sall = Sb, *Zall = Zc.p;
      long long ldU = ldn, ldS = ldsb, ldZ = ldn;
      DBuf<double> Uf, Sf, Zf;
      if (c->world > 1) {
        Uf.ensure(static_cast<size_t>(n));
        Sf.ensure(static_cast<size_t>(l) * n);
        Zf.ensure(static_cast<size_t>(l) * n);
        c->allgather_cols(U, ldn, 1, Uf.p, n);
        c->allgather_cols(Sb, ldsb, l, Sf.p, n);
        c->allgather_cols(Zc.p, ldn, l, Zf.p, n);
        Uall = Uf.p;
        Sall = Sf.p;
        Zall = Zf.p;
        ldU = ldS = ldZ = n;
      }
      conv(Uall, ldU, 1, Up);
      conv(Sall, ldS, l, SZp);
      conv(Zall, ldZ, l, SZp + elem * static_cast<size_t>(l) * n_pad);
      const void* Xp = fp64 ? static_cast<const void*>(c->X64s.p) : static_cast<const void*>(c->X32.p);
      int nblk = 0;
      const double cmix = static_cast<double>(n) / static_cast<double>(l);
      c->check_launch(gpk::launch_deriv_contract(fp64, c->family, c->dp, Xp, Up, SZp, r0, nl, n_pad, l, cmix, nullptr,
                                                 &nblk, c->st),
                      0, "deriv_contract");
      const int na = c->dp + 1;
      DBuf<double> part;
      part.ensure(static_cast<size_t>(nblk) * na);
      auto ev = c->prof_begin(1);
      c->check_launch(gpk::launch_deriv_contract(fp64, c->family, c->dp, Xp, Up, SZp, r0, nl, n_pad, l, cmix, part.p,
                                                 &nblk, c->st),
                      1, "deriv_contract");
      {
        const int cf[] = {2, 3, 6, 9};
        const double nn = static_cast<double>(nl) * n;
        c->prof_end(1, ev, nn * ((l + 1) + 2.0 * (d + 1) + 3.0 * d + cf[c->family] + 4.0), nn);
      }
      std::vector<double> hp(static_cast<size_t>(nblk) * na);
      c->d2h(hp.data(), part.p, sizeof(double) * hp.size());
      std::vector<double> tot(na, 0.0);
      for (int b = 0; b < nblk; ++b)
        for (int q = 0; q < na; ++q) tot[q] += hp[static_cast<size_t>(b) * na + q];
      tot = c->allreduce_host(tot);  // rank-ordered sum of the per-rank pair sums
      const double cpre = fp64 ? 1.0 : gpk::prescale_c(c->family);
      // outputscale: dK = 2 o shape ; lengthscale j: dK = (-2 o^2 / l_j) shape_ds ds_j^2;
      // tot[w] = quad[w] - (n/l) gamma[w] (raw), so the gradient is
      // 0.5 (quad - tdet - (n/l)(gamma - sum_i t_wi)) theta_w   (gp_likelihood.hpp:97-100)
      double mix[64];
      mix[0] = 2.0 * c->o * tot[0];
      for (int i = 0; i < l; ++i) zw[0][i] = std::nan("");
      per_probe[0] = false;
      for (int j = 0; j < d; ++j) {
        const double fac = (-2.0 * c->o2 / c->ls[j]) / cpre;
        mix[1 + j] = fac * tot[1 + j];
        per_probe[1 + j] = false;
      }
      c->entries += static_cast<long long>(nl) * n;
      for (int w = 0; w <= d; ++w) {
        double tsum = 0.0;
        for (int i = 0; i < l; ++i) tsum += tw[w][i];
        const double num = mix[w] - tdet[w] + static_cast<double>(n) / static_cast<double>(l) * tsum;
        res->gradient[w] = 0.5 * num * (w == 0 ? c->o : c->ls[w - 1]);
        if (res->backward_gammas && cfg->backward_mode != 3)
          for (int i = 0; i < l; ++i) res->backward_gammas[static_cast<size_t>(w) * l + i] = std::nan("");
      }
      if (res->backward_gammas && cfg->backward_mode == 3) {
        // per-probe backward gammas without the (d+1) l solves: z_i' K^-1 dK_w z_i = s_i' (dK_w z_i)
        // (K_hat^-1 symmetric, s_i the converged probe solves), one derivative MVM of the l
        // probes per parameter; gamma_i = s_i' dK_w z_i - z_i' P^-1 dP_w z_i
        // (trace_estimation.hpp:216-218)
        DBuf<double> RHw;
        RHw.ensure(static_cast<size_t>(l) * ldn);
        for (int w = 0; w <= d; ++w) {
          c->apply_kernel(Zc.p, ldn, l, RHw.p, ldn, fp64, w);
          const std::vector<double> zs = c->col_dots(Sb, RHw.p, l, ldn);
          for (int i = 0; i < l; ++i) res->backward_gammas[static_cast<size_t>(w) * l + i] = zs[i] - tw[w][i];
        }
      }
    } else {
      // reference-faithful: mBCG over the (d+1) l right-hand sides dK_w z_i (trace_estimation.hpp:209)
      const int tb = (d + 1) * l;
      DBuf<double> RH, Wsol;
      RH.ensure(static_cast<size_t>(tb) * ldn);
      Wsol.ensure(static_cast<size_t>(tb) * ldn);
      for (int w = 0; w <= d; ++w)
        c->apply_kernel(Zc.p, ldn, l, RH.p + static_cast<size_t>(w) * l * ldn, ldn, fp64, w);
      gpk_ctx::CgOut cgw;
      try {
        cgw = c->mbcg(RH.p, ldn, tb, mi, tol, fp64, Wsol.p, ldn, nullptr, nullptr, nullptr);
      } catch (const GpkError& e) {
        int col;
        const std::string m = strip_col(e.msg, &col);
        fail(GPK_NUMERICAL_ERROR, "trace residual: probe " + std::to_string(std::max(col, 0) % l) + ": " + m);
      }
      res->max_cg_rel_residual = std::max(res->max_cg_rel_residual, cgw.max_rel_pres());
      res->unconverged_columns += cgw.unconverged();
      if (!fp64 && cfg->solver.refine > 0) {
        double mr = -1.0;
        try {
          c->refine(RH.p, ldn, tb, Wsol.p, ldn, cgw, mi, tol, cfg->solver.refine, &mr);
        } catch (const GpkError& e) {
          int col;
          const std::string m = strip_col(e.msg, &col);
          fail(GPK_NUMERICAL_ERROR, "trace residual: probe " + std::to_string(std::max(col, 0) % l) + ": " + m);
        }
        res->max_true_rel_residual = std::max(res->max_true_rel_residual, mr);
      }
      for (int q = 0; q < tb; ++q) res->total_cg_iterations += cgw.iters[q];
      DBuf<double> du;
      du.ensure(static_cast<size_t>(ldn));
      for (int w = 0; w <= d; ++w) {
        const std::vector<double> zs = c->col_dots(Zc.p, Wsol.p + static_cast<size_t>(w) * l * ldn, l, ldn);
        for (int i = 0; i < l; ++i) zw[w][i] = zs[i];
        c->apply_kernel(U, ldn, 1, du.p, ldn, fp64, w);
        quadw[w] = c->col_dots(U, du.p, 1, ldn)[0];
      }
      for (int w = 0; w <= d; ++w) {
        std::vector<double> gm(l);
        double st = 0.0;
        for (int i = 0; i < l; ++i) {
          gm[i] = zw[w][i] - tw[w][i];  // gamma_i = z.(w - wt)
          st += gm[i];
        }
        st *= static_cast<double>(n) / static_cast<double>(l);
        const double tau = tdet[w] + st;
        res->gradient[w] = 0.5 * (quadw[w] - tau) * (w == 0 ? c->o : c->ls[w - 1]);
        if (res->backward_gammas)
          for (int i = 0; i < l; ++i) res->backward_gammas[static_cast<size_t>(w) * l + i] = gm[i];
      }
    }
    // noise component (gp_likelihood.hpp:87-101 with w = d+1)
    {
      const int w = d + 1;
      double st = 0.0;
      std::vector<double> gm(l);
      for (int i = 0; i < l; ++i) {
        gm[i] = zw[w][i] - tw[w][i];
        st += gm[i];
      }
      st *= static_cast<double>(n) / static_cast<double>(l);
      const double tau = tdet[w] + st;
      res->gradient[w] = 0.5 * (quadw[w] - tau) * c->noise;
      if (res->backward_gammas)
        for (int i = 0; i < l; ++i) res->backward_gammas[static_cast<size_t>(w) * l + i] = gm[i];
    }
  }
  CK(cudaEventRecord(e2, c->st));
  finish_forward();  // join the SLQ threads, finish the value (overlapped with the backward pass)
  c->sync();
  float ms1 = 0, ms2 = 0;
  CK(cudaEventElapsedTime(&ms1, e0, e1));
  CK(cudaEventElapsedTime(&ms2, e1, e2));
  res->seconds_solve = ms1 * 1e-3;
  res->seconds_backward = ms2 * 1e-3;
  res->seconds_total = (ms1 + ms2) * 1e-3;
  res->kernel_entries = c->entries;
  res->mvm_flops = c->flops;
  res->gpu_launches = static_cast<int>(c->launches - launches0);
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

const char* gpk_version(void) { return "gpkrylov_cuda 0.1 (sm_100a)"; }

gpk_status gpk_create(int device, gpk_ctx** out) {
  if (!out) return GPK_INPUT_ERROR;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return GPK_CUDA_ERROR;
  if (device < 0 || device >= ndev) return GPK_INPUT_ERROR;
  auto* c = new gpk_ctx();
  c->device = device;
  const gpk_status s = guard(c, [&] {
    CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = ~0ull;  // never trim: freed scratch is reused without synchronisation
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  });
  if (s != GPK_OK) {
    delete c;
    return s;
  }
  *out = c;
  return GPK_OK;
}

gpk_status gpk_nccl_unique_id(void* out) {
  if (!out) return GPK_INPUT_ERROR;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return GPK_NCCL_ERROR;
  std::memcpy(out, &id, sizeof(id));
  return GPK_OK;
}

gpk_status gpk_create_sharded(int device, int rank, int world, const void* nccl_id, gpk_ctx** out) {
  if (!out || !nccl_id || world < 1 || rank < 0 || rank >= world) return GPK_INPUT_ERROR;
  const gpk_status s0 = gpk_create(device, out);
  if (s0 != GPK_OK) return s0;
  gpk_ctx* c = *out;
  const gpk_status s = guard(c, [&] {
    auto nc = std::make_unique<NcclComm>();
    nc->rank = rank;
    nc->world = world;
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    const ncclResult_t r = ncclCommInitRank(&nc->c, world, id, rank);
    if (r != ncclSuccess) fail(GPK_NCCL_ERROR, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    c->comm = std::move(nc);
    c->rank = rank;
    c->world = world;
  });
  if (s != GPK_OK) {
    gpk_destroy(c);
    *out = nullptr;
  }
  return s;
}

gpk_status gpk_group_create(int world, gpk_group** out) {
  if (!out || world < 1) return GPK_INPUT_ERROR;
  auto* g = new gpk_group();
  g->world = world;
  g->host.resize(world);
  *out = g;
  return GPK_OK;
}

void gpk_group_destroy(gpk_group* g) { delete g; }

gpk_status gpk_create_in_group(int device, gpk_group* g, int rank, gpk_ctx** out) {
  if (!out || !g || rank < 0 || rank >= g->world) return GPK_INPUT_ERROR;
  const gpk_status s0 = gpk_create(device, out);
  if (s0 != GPK_OK) return s0;
  gpk_ctx* c = *out;
  auto gc = std::make_unique<GroupComm>();
  gc->g = g;
  gc->rank = rank;
  gc->world = g->world;
  c->comm = std::move(gc);
  c->rank = rank;
  c->world = g->world;
  return GPK_OK;
}

gpk_status gpk_shard_rows(const gpk_ctx* ctx, int64_t* r0, int64_t* r1) {
  if (!ctx || !r0 || !r1) return GPK_INPUT_ERROR;
  if (!ctx->have_data) return GPK_INPUT_ERROR;
  *r0 = ctx->r0;
  *r1 = ctx->r1;
  return GPK_OK;
}

void gpk_destroy(gpk_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->st);
  ctx->release_side();
  ctx->release_handles();
  for (auto& p : ctx->prof)
    for (auto& e : p.pending) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  cudaStream_t s = ctx->st;
  tl_stream = s;
  delete ctx;  // buffers return to the pool on their stream
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
}

const char* gpk_last_error(const gpk_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
long long gpk_launch_count(const gpk_ctx* ctx) { return ctx ? ctx->launches : 0; }
void* gpk_stream(const gpk_ctx* ctx) { return ctx ? static_cast<void*>(ctx->st) : nullptr; }

gpk_status gpk_set_mvm_variant(gpk_ctx* ctx, int variant) {
  return guard(ctx, [&] {
    require(variant >= GPK_MVM_AUTO && variant <= GPK_MVM_GRAM, "gpk_set_mvm_variant: unknown variant");
    ctx->mvm_variant = variant;
    ctx->packed = false;
  });
}
gpk_status gpk_get_mvm_variant(gpk_ctx* ctx, int* variant, double* max_sqnorm) {
  return guard(ctx, [&] {
    ctx->require_ready();
    if (variant) *variant = ctx->gram_ok ? GPK_MVM_GRAM : GPK_MVM_DIRECT;
    if (max_sqnorm) *max_sqnorm = ctx->gram_maxnorm;
  });
}

gpk_status gpk_profile_enable(gpk_ctx* ctx, int on) {
  return guard(ctx, [&] {
    ctx->prof_on = on != 0;
    ctx->prof_mask = on == 1 ? 3u : static_cast<unsigned>(on) & 15u;  // 1: kinds 0 and 1; else a mask
  });
}
gpk_status gpk_profile_read(gpk_ctx* ctx, int kind, double* ms, long long* launches, double* flops,
                            double* entries) {
  return guard(ctx, [&] {
    require(kind >= 0 && kind <= 3, "gpk_profile_read: kind must be 0..3");
    ctx->prof_collect();
    const auto& p = ctx->prof[kind];
    if (ms) *ms = p.ms;
    if (launches) *launches = p.launches;
    if (flops) *flops = p.fl;
    if (entries) *entries = p.en;
  });
}
gpk_status gpk_profile_reset(gpk_ctx* ctx) {
  return guard(ctx, [&] {
    ctx->prof_collect();
    for (auto& p : ctx->prof) {
      p.ms = p.fl = p.en = 0.0;
      p.launches = 0;
    }
  });
}

static void set_data_common(gpk_ctx* c, const double* X, int64_t n, int64_t d, int64_t ldx, bool device) {
  require(n >= 1, "KernelOperator: empty dataset");
  require(d >= 1, "Hyperparameters: need at least one lengthscale");
  require(ldx >= n, "gpk_set_data: ldx < n");
  require(gpk::dpad_for(static_cast<int>(d)) > 0, "gpkrylov_cuda: input dimension above 32 is not supported");
  require(n < (1LL << 30), "gpkrylov_cuda: n too large for one device");
  c->n = static_cast<int>(n);
  c->d = static_cast<int>(d);
  c->n_pad = static_cast<int>((n + 127) / 128 * 128);
  c->set_shard();  // this rank's rows [r0, r1) and the local leading dimension
  c->dp = gpk::dpad_for(c->d);
  c->X.ensure(static_cast<size_t>(n) * d);
  CK(cudaMemcpy2DAsync(c->X.p, n * sizeof(double), X, ldx * sizeof(double), n * sizeof(double), d,
                       device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->st));
  c->have_data = true;
  c->packed = false;
  c->pkind = 0;
  c->have_dl = false;
}

gpk_status gpk_set_data(gpk_ctx* ctx, const double* X, int64_t n, int64_t d, int64_t ldx) {
  return guard(ctx, [&] { set_data_common(ctx, X, n, d, ldx, false); ctx->sync(); });
}
gpk_status gpk_set_data_device(gpk_ctx* ctx, const double* dX, int64_t n, int64_t d, int64_t ldx) {
  return guard(ctx, [&] { set_data_common(ctx, dX, n, d, ldx, true); });
}

gpk_status gpk_set_params(gpk_ctx* ctx, int family, double alpha, double log_o, const double* log_ls,
                          double log_noise) {
  return guard(ctx, [&] {
    (void)alpha;
    require(family >= 0 && family <= 4, "KernelSpec: unknown kernel family");
    require(family != GPK_RATQUAD, "gpkrylov_cuda: rational quadratic kernel is not supported on the GPU path");
    require(ctx->have_data, "gpkrylov_cuda: set data before hyperparameters");
    auto ok = [](double lv) { return std::isfinite(lv) && std::isfinite(std::exp(lv)) && std::exp(lv) > 0.0; };
    require(ok(log_o), "Hyperparameters: output scale not positive finite");  // kernels.hpp:55-63
    require(ok(log_noise), "Hyperparameters: noise variance not positive finite");
    for (int j = 0; j < ctx->d; ++j)
      require(ok(log_ls[j]), "Hyperparameters: lengthscale " + std::to_string(j) + " not positive finite");
    ctx->family = family;
    ctx->log_o = log_o;
    ctx->log_noise = log_noise;
    ctx->log_ls.assign(log_ls, log_ls + ctx->d);
    ctx->o = std::exp(log_o);
    ctx->o2 = std::pow(ctx->o, 2);
    ctx->noise = std::exp(log_noise);
    ctx->ls.resize(ctx->d);
    for (int j = 0; j < ctx->d; ++j) ctx->ls[j] = std::exp(log_ls[j]);
    ctx->have_params = true;
    ctx->packed = false;
    ctx->pack();
  });
}

static void mvm_common(gpk_ctx* c, int which, const double* V, int64_t ldv, int t, double* out, int64_t ldo,
                       int precision) {
  c->require_ready();
  require(t >= 1, "KernelOperator: vector length does not match n");
  require(which >= -1 && which <= c->d + 1, "KernelOperator: hyperparameter index out of range");
  const int n = c->n;
  for (int q = 0; q < t; ++q)
    for (int i = 0; i < n; ++i)
      if (!std::isfinite(V[q * ldv + i])) fail(GPK_INPUT_ERROR, "KernelOperator: non-finite entries in input vector");
  require(precision >= GPK_PREC_FP64 && precision <= GPK_PREC_TF32X3, "gpk_kernel_mvm: unknown precision");
  c->use_tc = precision == GPK_PREC_TF32X3;
  DBuf<double> dv, dout;
  dv.ensure(static_cast<size_t>(t) * c->ldn);
  dout.ensure(static_cast<size_t>(t) * c->ldn);
  // sharded: this rank uploads and writes back its rows [r0, r1) only
  const int nl = c->nl, r0 = c->r0;
  CK(cudaMemcpy2DAsync(dv.p, c->ldn * sizeof(double), V + r0, ldv * sizeof(double), nl * sizeof(double), t,
                       cudaMemcpyHostToDevice, c->st));
  c->apply_kernel(dv.p, c->ldn, t, dout.p, c->ldn, precision == GPK_PREC_FP64, which);
  if (which < 0) c->check_launch(gpk::launch_axpby(dout.p, dv.p, 1.0, c->noise, nl, t, c->ldn, c->st), 1, "axpy");
  CK(cudaMemcpy2DAsync(out + r0, ldo * sizeof(double), dout.p, c->ldn * sizeof(double), nl * sizeof(double), t,
                       cudaMemcpyDeviceToHost, c->st));
  c->sync();
}

gpk_status gpk_kernel_mvm(gpk_ctx* ctx, const double* V, int64_t ldv, int t, double* out, int64_t ldo, int precision) {
  return guard(ctx, [&] { mvm_common(ctx, -1, V, ldv, t, out, ldo, precision); });
}
gpk_status gpk_kernel_deriv_mvm(gpk_ctx* ctx, int which, const double* V, int64_t ldv, int t, double* out,
                                int64_t ldo, int precision) {
  return guard(ctx, [&] {
    if (which < 0 || which > ctx->d + 1) fail(GPK_INPUT_ERROR, "KernelOperator: hyperparameter index out of range");
    mvm_common(ctx, which, V, ldv, t, out, ldo, precision);
  });
}

static void column_common(gpk_ctx* c, int which, int64_t i, double* out) {
  c->require_ready();
  require(i >= 0 && i < c->n, which < 0 ? "kernel_column: index out of range" : "kernel_deriv_column: index out of range");
  require(which >= -1 && which <= c->d + 1, "KernelOperator: hyperparameter index out of range");
  DBuf<double> col;
  col.ensure(c->n);
  if (which == c->d + 1) {
    std::fill(out, out + c->n, 0.0);
    return;
  }
  double fac = 1.0;
  if (which == 0) fac = 2.0 / c->o;
  if (which >= 1) {
    const double lj = c->ls[which - 1];
    fac = -2.0 * c->o2 / (lj * lj * lj);
  }
  c->check_launch(gpk::launch_kernel_column(c->family, c->sx.p, c->X.p, c->sq.p, c->n, c->d, i, which, c->o2, fac,
                                            col.p, c->st),
                  1, "kernel_column");
  c->d2h(out, col.p, sizeof(double) * c->n);
}

gpk_status gpk_kernel_column(gpk_ctx* ctx, int64_t i, double* out) {
  return guard(ctx, [&] { column_common(ctx, -1, i, out); });
}
gpk_status gpk_kernel_deriv_column(gpk_ctx* ctx, int which, int64_t i, double* out) {
  return guard(ctx, [&] {
    if (which < 0 || which > ctx->d + 1) fail(GPK_INPUT_ERROR, "KernelOperator: hyperparameter index out of range");
    column_common(ctx, which, i, out);
  });
}

gpk_status gpk_precond_identity(gpk_ctx* ctx) {
  return guard(ctx, [&] {
    require(ctx->have_data, "gpkrylov_cuda: no data set (gpk_set_data)");
    ctx->pkind = 1;
    ctx->k = 0;
    ctx->plogdet = 0.0;
    ctx->have_dl = true;
    ctx->trace_det.assign(ctx->d + 2, 0.0);
    ctx->trace_pending = false;  // a new preconditioner: no derivative traces pending
  });
}

// preconditioners.hpp:236-264 + DiagPlusLowRank ctor (:84-95)
gpk_status gpk_pivoted_cholesky(gpk_ctx* ctx, int rank, double diag_tol, double noise, int64_t* pivots_out,
                                int* achieved, double* remaining_diag) {
  return guard(ctx, [&] {
    gpk_ctx* c = ctx;
    c->require_ready();
    const int n = c->n;
    require(rank >= 0 && rank <= n, "pivoted_cholesky: rank must be in [0, n]");
    require(noise > 0.0 && std::isfinite(noise), "DiagPlusLowRank: noise variance must be positive");
    c->pkind = 0;
    c->have_dl = false;
    c->pivots.clear();
    const bool shard = c->world > 1;
    const int nrow = shard ? c->nl : n;  // rows of the diagonal / factor this rank computes
    c->pshard = shard;
    c->ldP = shard ? static_cast<long long>(c->nl) + rank : n;  // sharded: own rows, then the pivot rows
    DBuf<double> dg, col;
    dg.ensure(nrow);
    col.ensure(n);
    c->L.ensure(static_cast<size_t>(c->ldP) * std::max(rank, 1));
    const long long cnt = nrow;
    fill_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, c->st>>>(dg.p, cnt, c->o * c->o);  // :230-233
    c->check_launch(cudaGetLastError(), 1, "fill");
    const double kmax = c->o * c->o;
    const int nb = gpk::pchol_blocks(n);
    c->w_argval.ensure(nb + 1);
    c->w_argidx.ensure(nb + 1);
    // the whole factorisation is enqueued at once; the pivot (argmax, lowest index on
    // ties) and the stopping rules (:250-253) live in a device-resident state
    int step = 0;
    if (shard && rank > 0 && !(kmax <= diag_tol)) {
      // row-sharded: per-step kernels on the own rows, candidates and pivot rows all-gathered
      // (gpk_pchol.cu); no host round trip until the end
      DBuf<gpk::PivotState> ps;
      DBuf<long long> dpiv;
      DBuf<double> lp, cand, cands, rows, rowsr;
      ps.ensure(1);
      dpiv.ensure(rank);
      lp.ensure(rank);
      cand.ensure(2);
      cands.ensure(2 * static_cast<size_t>(c->world));
      rows.ensure(rank);
      rowsr.ensure(static_cast<size_t>(rank) * c->world);
      gpk::PivotState h0{};
      h0.dp = kmax;
      h0.p = 0;
      c->h2d(ps.p, &h0, sizeof(h0));
      const int grid = gpk::pchol_shard_grid(c->nl);
      c->w_argval.ensure(grid);
      c->w_argidx.ensure(grid);
      for (int st_ = 0; st_ < rank; ++st_) {
        c->check_launch(gpk::launch_pchol_shard_step(c->family, c->sx.p, c->sq.p, n, c->d, c->o2, c->L.p, c->ldP,
                                                     c->r0, c->nl, st_, lp.p, ps.p, dg.p, c->w_argval.p,
                                                     c->w_argidx.p, grid, cand.p, c->st),
                        2, "pchol_shard_step");
        c->comm->allgather(cand.p, cands.p, 2 * sizeof(double), c->st);
        c->check_launch(gpk::launch_pchol_shard_select(cands.p, c->world, st_, diag_tol, kmax, ps.p, dpiv.p, c->L.p,
                                                       c->ldP, c->r0, c->nl, rank, rows.p, c->st),
                        2, "pchol_shard_select");
        if (st_ + 1 < rank) {
          c->comm->allgather(rows.p, rowsr.p, sizeof(double) * rank, c->st);
          c->check_launch(gpk::launch_pchol_shard_rowtake(rowsr.p, c->world, rank, c->d_r0.p, c->d_rows.p, ps.p, lp.p,
                                                          c->st),
                          1, "pchol_shard_rowtake");
        }
      }
      gpk::PivotState hs{};
      c->d2h(&hs, ps.p, sizeof(hs));
      step = hs.done;
      if (hs.negative)
        fail(GPK_NUMERICAL_ERROR, "pivoted_cholesky: negative pivot " + num(hs.dp) + " at step " +
                                      std::to_string(step) + "; matrix not PSD");
      c->pivots.resize(step);
      if (step > 0) c->d2h(c->pivots.data(), dpiv.p, sizeof(long long) * step);
      // the pivot rows L[p_q, :] (owned by one rank each) appended as rows nl .. nl + k - 1
      if (step > 0) {
        DBuf<double> pr, prr;
        pr.ensure(static_cast<size_t>(rank) * rank);
        prr.ensure(static_cast<size_t>(rank) * rank * c->world);
        c->check_launch(gpk::launch_pchol_pivot_rows(0, c->L.p, pr.p, c->ldP, c->r0, c->nl, rank, dpiv.p, c->world,
                                                     c->d_r0.p, c->d_rows.p, c->st),
                        1, "pivot_rows");
        c->comm->allgather(pr.p, prr.p, sizeof(double) * rank * rank, c->st);
        c->check_launch(gpk::launch_pchol_pivot_rows(1, prr.p, c->L.p, c->ldP, c->r0, c->nl, rank, dpiv.p, c->world,
                                                     c->d_r0.p, c->d_rows.p, c->st),
                        1, "pivot_rows");
      }
    } else if (!shard && rank > 0 && !(kmax <= diag_tol)) {  // step 0: diagonal o^2, pivot 0
      DBuf<gpk::PivotState> ps;
      DBuf<long long> dpiv;
      ps.ensure(1);
      dpiv.ensure(rank);
      gpk::PivotState h0{};
      h0.dp = kmax;
      h0.p = 0;
      c->h2d(ps.p, &h0, sizeof(h0));
      // one cooperative launch for all steps (gpk_pchol.cu); the per-step kernels remain the
      // fallback when the pivot row does not fit in shared memory or co-residency is unavailable
      const size_t psm = sizeof(double) * static_cast<size_t>(rank);
      const int pg = (psm <= 200 * 1024 && c->use_persistent_pchol) ? gpk::pchol_persistent_grid(n, psm) : 0;
      if (pg > 0) {
        c->w_argval.ensure(2 * static_cast<size_t>(pg) + 1);
        c->w_argidx.ensure(2 * static_cast<size_t>(pg) + 1);
        c->check_launch(gpk::launch_pchol_persistent(c->family, c->sx.p, c->sq.p, n, c->d, c->o2, c->L.p, rank,
                                                     diag_tol, kmax, dg.p, c->w_argval.p, c->w_argidx.p, ps.p,
                                                     dpiv.p, pg, c->st),
                        1, "pivoted_cholesky");
      } else {
        c->check_launch(gpk::launch_pchol_dev(c->family, c->sx.p, c->sq.p, n, c->d, c->o2, c->L.p, rank, diag_tol,
                                              kmax, col.p, dg.p, c->w_argval.p, c->w_argidx.p, ps.p, dpiv.p, c->st),
                        3 * rank, "pivoted_cholesky");
      }
      gpk::PivotState hs{};
      c->d2h(&hs, ps.p, sizeof(hs));
      step = hs.done;  // steps whose column was produced
      if (hs.negative)
        fail(GPK_NUMERICAL_ERROR, "pivoted_cholesky: negative pivot " + num(hs.dp) + " at step " +
                                      std::to_string(step) + "; matrix not PSD");
      c->pivots.resize(step);
      if (step > 0) c->d2h(c->pivots.data(), dpiv.p, sizeof(long long) * step);
    }
    c->k = step;
    if (achieved) *achieved = step;
    if (pivots_out)
      for (int s = 0; s < step; ++s) pivots_out[s] = c->pivots[s];
    if (remaining_diag) {
      if (shard) {
        DBuf<double> full;
        full.ensure(n);
        c->allgather_cols(dg.p, nrow, 1, full.p, n);
        c->d2h(remaining_diag, full.p, sizeof(double) * n);
      } else {
        c->d2h(remaining_diag, dg.p, sizeof(double) * n);
      }
    }
    // DiagPlusLowRank (:84-95): inner = L'L + s2 I, Cholesky inner = R R', C = L inner^{-1}
    // = (L R^-T) R^-1, log det P (:127-133) -- k x k work on the device (cuBLAS/cuSOLVER)
    c->pnoise = noise;
    const int k = c->k;
    double ld = static_cast<double>(n) * std::log(noise);
    if (k > 0) {
      c->ensure_handles();
      DBuf<double> G;
      DBuf<int> info;
      G.ensure(static_cast<size_t>(k) * k);
      info.ensure(1);
      const double one = 1.0, zero = 0.0;
      CB(cublasDsyrk(c->blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, k, nrow, &one, c->L.p, c->ldP, &zero, G.p, k));
      if (shard) c->allreduce_sum(G.p, static_cast<long long>(k) * k);  // L'L over all rows, rank order
      add_diag_kernel<<<(k + 255) / 256, 256, 0, c->st>>>(G.p, k, noise);
      c->check_launch(cudaGetLastError(), 2, "gram");
      int lwork = 0;
      CS(cusolverDnDpotrf_bufferSize(c->solver, CUBLAS_FILL_MODE_LOWER, k, G.p, k, &lwork));
      DBuf<double> work;
      work.ensure(static_cast<size_t>(std::max(lwork, 1)));
      CS(cusolverDnDpotrf(c->solver, CUBLAS_FILL_MODE_LOWER, k, G.p, k, work.p, lwork, info.p));
      int hinfo = 0;
      std::vector<double> diag(k);
      CK(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpy2DAsync(diag.data(), sizeof(double), G.p, (k + 1) * sizeof(double), sizeof(double), k,
                           cudaMemcpyDeviceToHost, c->st));
      c->sync();  // one round trip for the factorisation status and the diagonal
      if (hinfo != 0)
        fail(GPK_NUMERICAL_ERROR, "DiagPlusLowRank: inner Cholesky failed (cannot happen for sigma^2 > 0)");
      double sl = 0.0;
      for (int a = 0; a < k; ++a) sl += std::log(diag[a]);
      ld += 2.0 * sl - static_cast<double>(k) * std::log(noise);
      c->C.ensure(static_cast<size_t>(c->ldP) * k);
      CK(cudaMemcpyAsync(c->C.p, c->L.p, sizeof(double) * static_cast<size_t>(c->ldP) * k, cudaMemcpyDeviceToDevice,
                         c->st));
      CB(cublasDtrsm(c->blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, nrow, k,
                     &one, G.p, k, c->C.p, c->ldP));
      CB(cublasDtrsm(c->blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, nrow, k,
                     &one, G.p, k, c->C.p, c->ldP));
      c->launches += 4;
      // G and work are released stream-ordered; C is consumed on the same stream
    }
    c->plogdet = ld;
    c->pkind = 2;
    // trace of P^{-1} for the noise derivative: (n - sum C o L) / s2  (:138-145 with dP = I)
    c->trace_det.assign(c->d + 2, 0.0);
    c->trace_pending = false;  // a new preconditioner: no derivative traces pending
    double cl = 0.0;
    if (k > 0 && shard) {
      const std::vector<double> cd = c->col_dots(c->C.p, c->L.p, k, c->ldP);  // own rows, rank-order sum
      for (int q = 0; q < k; ++q) cl += cd[q];
    } else if (k > 0) {
      const int nrb = gpk::num_chunks(n * k);
      DBuf<double> part, outv;
      part.ensure(nrb);
      outv.ensure(1);
      // flat dot over n*k entries
      c->check_launch(gpk::launch_dot_partials(0, c->C.p, c->L.p, 0.0, n * k, 0, 1, part.p, c->st), 1, "dot");
      c->check_launch(gpk::launch_reduce_partials(part.p, nrb, 1, outv.p, c->st), 1, "reduce");
      c->d2h(&cl, outv.p, sizeof(double));
    }
    c->trace_det[c->d + 1] = static_cast<double>(n) / noise - cl / noise;
  });
}

// preconditioners.hpp:269-295
gpk_status gpk_precond_deriv_factors(gpk_ctx* ctx) {
  return guard(ctx, [&] {
    gpk_ctx* c = ctx;
    c->require_ready();
    if (c->pkind == 1) return;
    require(c->pkind == 2, "DiagPlusLowRank: derivative factors not attached");
    const int n = c->n, k = c->k, nw = c->d + 1;
    require(static_cast<int>(c->pivots.size()) == k,
            "pivoted_cholesky_deriv_factors: preconditioner has no pivot record");
    c->have_dl = false;
    if (k > 0) {
      // rows of the recursion: all n (unsharded), or -- row-sharded -- the own rows followed by
      // the k pivot rows (the only rows another row's recursion reads), so every rank builds
      // the factors of exactly the rows it owns: the reference's algorithm on that row set
      const bool shard = c->pshard;
      const int N = shard ? static_cast<int>(c->ldP) : n;
      DBuf<double> xs_e, x_e, sq_e;
      DBuf<long long> piv_e;
      c->dL.ensure(static_cast<size_t>(nw) * N * k);
      c->w_trace.ensure(nw);
      // the build runs on the side stream st2 (fork after L, pivots and dL's allocation on st);
      // its scratch is allocated and released on st2 (sharded: on st, its traces are all-reduced)
      cudaStream_t ds = c->st;
      if (c->use_side && !shard) {
        c->ensure_side();
        ds = c->st2;
        CK(cudaEventRecord(c->ev_fork, c->st));
        CK(cudaStreamWaitEvent(ds, c->ev_fork, 0));
        tl_stream = ds;
      }
      struct StreamRestore {
        gpk_ctx* c;
        ~StreamRestore() {
          tl_stream = c->st;
          if (c->blas) cublasSetStream(c->blas, c->st);
        }
      } restore{c};
      DBuf<double> facs;
      facs.ensure(nw);
      std::vector<double> hf(nw);
      for (int w = 0; w < nw; ++w) {  // kernels.hpp:262 (outputscale) and :270-272 (lengthscales)
        hf[w] = 2.0 / c->o;
        if (w >= 1) {
          const double lj = c->ls[w - 1];
          hf[w] = -2.0 * c->o2 / (lj * lj * lj);
        }
      }
      CK(cudaMemcpyAsync(facs.p, hf.data(), sizeof(double) * nw, cudaMemcpyHostToDevice, ds));
      // Left-looking blocks of kB columns: the contribution of all earlier columns to a block is two
      // strided-batched GEMMs over the parameters, the recursion inside the block one kernel per column
      // (same formula as preconditioners.hpp:283-290, summation regrouped by block).
      constexpr int kB = 32;
      const long long wstride = static_cast<long long>(N) * k;
      DBuf<double> DC, Lp, dLp;
      DBuf<long long> dpiv;
      DC.ensure(static_cast<size_t>(nw) * N * kB);
      Lp.ensure(static_cast<size_t>(k) * kB);
      dLp.ensure(static_cast<size_t>(nw) * k * kB);
      dpiv.ensure(k);
      CK(cudaMemcpyAsync(dpiv.p, c->pivots.data(), sizeof(long long) * k, cudaMemcpyHostToDevice, ds));
      const double* sxp = c->sx.p;
      const double* xp = c->X.p;
      const double* sqp = c->sq.p;
      const long long* pivp = dpiv.p;
      if (shard) {  // coordinates of the extended rows; pivot q is row nl + q
        xs_e.ensure(static_cast<size_t>(c->d) * N);
        x_e.ensure(static_cast<size_t>(c->d) * N);
        sq_e.ensure(N);
        piv_e.ensure(k);
        c->check_launch(gpk::launch_gather_ext_rows(c->sx.p, n, c->d, c->r0, c->nl, dpiv.p, k, xs_e.p, N, ds), 1,
                        "ext_rows");
        c->check_launch(gpk::launch_gather_ext_rows(c->X.p, n, c->d, c->r0, c->nl, dpiv.p, k, x_e.p, N, ds), 1,
                        "ext_rows");
        c->check_launch(gpk::launch_gather_ext_rows(c->sq.p, n, 1, c->r0, c->nl, dpiv.p, k, sq_e.p, N, ds), 1,
                        "ext_rows");
        c->check_launch(gpk::launch_iota_ll(piv_e.p, k, c->nl, ds), 1, "iota");
        sxp = xs_e.p;
        xp = x_e.p;
        sqp = sq_e.p;
        pivp = piv_e.p;
      }
      DBuf<double> rep;
      rep.ensure(gpk::dl_replay_workspace(nw));
      c->ensure_handles();
      CB(cublasSetStream(c->blas, ds));
      for (int s0 = 0; s0 < k; s0 += kB) {
        const int bb = std::min(kB, k - s0);
        // DC_w[:, q] = dK_w column of pivot s0+q (all pivots of the block in one launch)
        c->check_launch(gpk::launch_deriv_columns_block(c->family, sxp, xp, sqp, N, c->d, pivp + s0, bb,
                                                        nw, facs.p, c->o2, DC.p, static_cast<long long>(N) * kB,
                                                        ds),
                        1, "deriv_columns_block");
        if (s0 > 0) {
          // Lp[c][q] = L[piv_q, c], dLp_w[c][q] = dL_w[piv_q, c]   (s0 x bb, column-major)
          c->check_launch(gpk::launch_gather_pivot_rows(c->L.p, N, 0, 1, pivp + s0, s0, bb, Lp.p, ds), 1,
                          "gather_pivot_rows");
          c->check_launch(gpk::launch_gather_pivot_rows(c->dL.p, N, wstride, nw, pivp + s0, s0, bb, dLp.p, ds),
                          1, "gather_pivot_rows");
          const double m1 = -1.0, one = 1.0;
          // DC_w -= dL_w[:, :s0] Lp ;  DC_w -= L[:, :s0] dLp_w
          CB(cublasDgemmStridedBatched(c->blas, CUBLAS_OP_N, CUBLAS_OP_N, N, bb, s0, &m1, c->dL.p, N, wstride, Lp.p,
                                       s0, 0, &one, DC.p, N, static_cast<long long>(N) * kB, nw));
          CB(cublasDgemmStridedBatched(c->blas, CUBLAS_OP_N, CUBLAS_OP_N, N, bb, s0, &m1, c->L.p, N, 0, dLp.p, s0,
                                       static_cast<long long>(s0) * bb, &one, DC.p, N,
                                       static_cast<long long>(N) * kB, nw));
          c->launches += 2;
        }
        // in-block recursion: one launch per block (every CTA replays the pivot rows' recursion)
        c->check_launch(gpk::launch_dl_block(c->L.p, c->dL.p, wstride, nw, s0, bb, pivp + s0, DC.p,
                                             static_cast<long long>(N) * kB, N, rep.p, ds),
                        2, "dl_block");
      }
      // tr(P^{-1} dP_w) = 2 sum(C o dL_w)  (algebraically equal to preconditioners.hpp:138-145)
      // all nw traces on the device; the host reads them when it needs them (need_trace)
      if (shard) {  // own rows per rank, rank-ordered sums
        std::vector<double> tr(nw, 0.0);
        for (int w = 0; w < nw; ++w) {
          const std::vector<double> cd = c->col_dots(c->C.p, c->dL.p + static_cast<size_t>(w) * N * k, k, N);
          for (int q = 0; q < k; ++q) tr[w] += cd[q];
        }
        c->h2d(c->w_trace.p, tr.data(), sizeof(double) * nw);
        c->trace_pending = true;
        c->have_dl = true;
        return;
      }
      const int nrb = gpk::num_chunks(n * k);
      DBuf<double> part;
      part.ensure(static_cast<size_t>(nrb) * nw);
      for (int w = 0; w < nw; ++w) {
        c->check_launch(gpk::launch_dot_partials(0, c->C.p, c->dL.p + static_cast<size_t>(w) * n * k, 0.0, n * k, 0, 1,
                                                 part.p + static_cast<size_t>(w) * nrb, ds),
                        1, "dot");
        c->check_launch(gpk::launch_reduce_partials(part.p + static_cast<size_t>(w) * nrb, nrb, 1, c->w_trace.p + w,
                                                    ds),
                        1, "reduce");
      }
      c->trace_pending = true;
      if (c->use_side) {
        CK(cudaEventRecord(c->ev_dl, ds));
        c->dl_pending = true;
      }
    }
    c->have_dl = true;
  });
}

gpk_status gpk_precond_factor(gpk_ctx* ctx, double* L, int64_t ldl) {
  return guard(ctx, [&] {
    require(ctx->pkind == 2, "gpkrylov_cuda: no pivoted-Cholesky preconditioner");
    if (ctx->k == 0) return;
    const double* src = ctx->L.p;
    DBuf<double> full;
    if (ctx->pshard) {  // every rank's own rows, gathered
      full.ensure(static_cast<size_t>(ctx->n) * ctx->k);
      ctx->allgather_cols(ctx->L.p, ctx->ldP, ctx->k, full.p, ctx->n);
      src = full.p;
    }
    CK(cudaMemcpy2DAsync(L, ldl * sizeof(double), src, ctx->n * sizeof(double), ctx->n * sizeof(double), ctx->k,
                         cudaMemcpyDeviceToHost, ctx->st));
    ctx->sync();
  });
}

gpk_status gpk_precond_deriv_factor(gpk_ctx* ctx, int which, double* dL, int64_t ldl) {
  return guard(ctx, [&] {
    require(ctx->pkind == 2 && ctx->have_dl, "DiagPlusLowRank: derivative factors not attached");
    require(which >= 0 && which <= ctx->d + 1, "DiagPlusLowRank: hyperparameter index out of range");
    const int n = ctx->n, k = ctx->k;
    if (k == 0) return;
    if (which == ctx->d + 1) {
      for (int c = 0; c < k; ++c) std::fill(dL + c * ldl, dL + c * ldl + n, 0.0);
      return;
    }
    const double* src = ctx->dL.p + static_cast<size_t>(which) * ctx->ldP * k;
    DBuf<double> full;
    if (ctx->pshard) {  // every rank's own rows, gathered
      full.ensure(static_cast<size_t>(n) * k);
      ctx->allgather_cols(src, ctx->ldP, k, full.p, n);
      src = full.p;
    }
    CK(cudaMemcpy2DAsync(dL, ldl * sizeof(double), src, n * sizeof(double), n * sizeof(double), k,
                         cudaMemcpyDeviceToHost, ctx->st));
    ctx->sync();
  });
}

gpk_status gpk_precond_solve(gpk_ctx* ctx, const double* V, int64_t ldv, int t, double* out, int64_t ldo) {
  return guard(ctx, [&] {
    require(ctx->pkind != 0, "gpkrylov_cuda: no preconditioner");
    const int nl = ctx->nl, r0 = ctx->r0;  // sharded: own rows only
    DBuf<double> dv, dz;
    dv.ensure(static_cast<size_t>(t) * ctx->ldn);
    dz.ensure(static_cast<size_t>(t) * ctx->ldn);
    CK(cudaMemcpy2DAsync(dv.p, ctx->ldn * sizeof(double), V + r0, ldv * sizeof(double), nl * sizeof(double), t,
                         cudaMemcpyHostToDevice, ctx->st));
    ctx->psolve(dv.p, t, dz.p);
    CK(cudaMemcpy2DAsync(out + r0, ldo * sizeof(double), dz.p, ctx->ldn * sizeof(double), nl * sizeof(double), t,
                         cudaMemcpyDeviceToHost, ctx->st));
    ctx->sync();
  });
}

gpk_status gpk_precond_logdet(gpk_ctx* ctx, double* out) {
  return guard(ctx, [&] {
    require(ctx->pkind != 0, "gpkrylov_cuda: no preconditioner");
    *out = ctx->pkind == 1 ? 0.0 : ctx->plogdet;
  });
}

gpk_status gpk_precond_trace_inv_deriv(gpk_ctx* ctx, int which, double* out) {
  return guard(ctx, [&] {
    require(ctx->pkind != 0, "gpkrylov_cuda: no preconditioner");
    require(which >= 0 && which <= ctx->d + 1, "DiagPlusLowRank: hyperparameter index out of range");
    if (ctx->pkind == 1) {
      *out = 0.0;
      return;
    }
    if (which <= ctx->d && ctx->k > 0) require(ctx->have_dl, "DiagPlusLowRank: derivative factors not attached");
    ctx->need_trace();
    *out = ctx->trace_det[which];
  });
}

gpk_status gpk_mbcg(gpk_ctx* ctx, const double* B, int64_t ldb, int t, const gpk_cg_cfg* cfg, double* X, int64_t ldx,
                    int* iters, int* converged, double* alpha, double* beta, double* resid_hist) {
  return guard(ctx, [&] {
    gpk_ctx* c = ctx;
    c->require_ready();
    require(cfg != nullptr, "gpk_mbcg: null config");
    require(c->pkind != 0, "gpkrylov_cuda: no preconditioner");
    require(t >= 1, "batched_pcg: rhs rows do not match operator");
    require(cfg->max_iters >= 1, "CgConfig: max_iters must be >= 1");
    require(cfg->rel_tol > 0.0 && cfg->rel_tol < 1.0, "CgConfig: rel_tol must be in (0, 1)");
    const int n = c->n;
    for (int q = 0; q < t; ++q)
      for (int i = 0; i < n; ++i)
        if (!std::isfinite(B[q * ldb + i])) fail(GPK_INPUT_ERROR, "KernelOperator: non-finite entries in input vector");
    const int mi = cfg->max_iters;
    DBuf<double> db, dx;
    db.ensure(static_cast<size_t>(t) * c->ldn);
    dx.ensure(static_cast<size_t>(t) * c->ldn);
    // sharded: this rank solves for its rows [r0, r1) of every column
    CK(cudaMemcpy2DAsync(db.p, c->ldn * sizeof(double), B + c->r0, ldb * sizeof(double), c->nl * sizeof(double), t,
                         cudaMemcpyHostToDevice, c->st));
    require(cfg->precision >= GPK_PREC_FP64 && cfg->precision <= GPK_PREC_TF32X3, "CgConfig: unknown precision");
    const bool fp64 = cfg->precision == GPK_PREC_FP64;
    c->use_tc = cfg->precision == GPK_PREC_TF32X3;
    gpk_ctx::CgOut r;
    try {
      r = c->mbcg(db.p, c->ldn, t, mi, cfg->rel_tol, fp64, dx.p, c->ldn, alpha, beta, resid_hist);
    } catch (const GpkError& e) {
      int col;
      const std::string m = strip_col(e.msg, &col);
      fail(GPK_SOLVER_ERROR, "batched_pcg: column " + std::to_string(col) + ": " + m);  // krylov.hpp:149-151
    }
    if (!fp64 && cfg->refine > 0) {
      double mr;
      c->refine(db.p, c->ldn, t, dx.p, c->ldn, r, mi, cfg->rel_tol, cfg->refine, &mr);
    }
    CK(cudaMemcpy2DAsync(X + c->r0, ldx * sizeof(double), dx.p, c->ldn * sizeof(double), c->nl * sizeof(double), t,
                         cudaMemcpyDeviceToHost, c->st));
    c->sync();
    for (int q = 0; q < t; ++q) {
      if (iters) iters[q] = r.iters[q];
      if (converged) converged[q] = r.converged[q];
    }
  });
}

gpk_status gpk_evaluate_mll_device(gpk_ctx* ctx, const double* dy, const double* dZ, int64_t ldz, int l,
                                   uint64_t probe_seed, const gpk_mll_cfg* cfg, gpk_mll_result* res) {
  return guard(ctx, [&] { evaluate_impl(ctx, dy, dZ, ldz, l, probe_seed, cfg, res); }, true);
}

gpk_status gpk_evaluate_mll(gpk_ctx* ctx, const double* y, const double* Z, int64_t ldz, int l, uint64_t probe_seed,
                            const gpk_mll_cfg* cfg, gpk_mll_result* res) {
  return guard(ctx, [&] {
    gpk_ctx* c = ctx;
    c->require_ready();
    require(l >= 1, "make_probes: need at least one probe");
    const int n = c->n;
    for (int i = 0; i < n; ++i)
      if (!std::isfinite(y[i])) fail(GPK_INPUT_ERROR, "KernelOperator: non-finite entries in input vector");
    DBuf<double> dy, dz;
    dy.ensure(n);
    dz.ensure(static_cast<size_t>(l) * n);
    c->h2d(dy.p, y, sizeof(double) * n);
    CK(cudaMemcpy2DAsync(dz.p, n * sizeof(double), Z, ldz * sizeof(double), n * sizeof(double), l,
                         cudaMemcpyHostToDevice, c->st));
    evaluate_impl(c, dy.p, dz.p, n, l, probe_seed, cfg, res);
  }, true);
}

// ---- validation / test metric and predictive mean ------------------

// mll_exact (gp_likelihood.hpp:124-146) on the device: dense K_hat in fp64 (the
// reference's expanded distances), cuSOLVER Cholesky, log det from its diagonal;
// the gradient from K_hat^{-1} (potri) contracted with each dense dK_w.
gpk_status gpk_mll_exact(gpk_ctx* ctx, const double* y, double* value, double* gradient) {
  return guard(ctx, [&] {
    gpk_ctx* c = ctx;
    c->require_ready();
    require(c->world == 1, "mll_exact: not available on a row-sharded context");
    require(value != nullptr, "mll_exact: null output");
    const int n = c->n;
    require(static_cast<double>(n) * n * 8.0 * (gradient ? 2.0 : 1.0) <= 96e9,
            "mll_exact: n too large for a dense factorisation");
    for (int i = 0; i < n; ++i)
      if (!std::isfinite(y[i])) fail(GPK_INPUT_ERROR, "KernelOperator: non-finite entries in input vector");
    c->ensure_handles();
    DBuf<double> K, a, work, part;
    DBuf<int> info;
    K.ensure(static_cast<size_t>(n) * n);
    a.ensure(n);
    part.ensure(n);
    info.ensure(1);
    c->check_launch(gpk::launch_dense_kernel(c->family, c->sx.p, c->X.p, c->sq.p, n, c->d, -1, c->o2, 1.0, K.p, n,
                                             c->st),
                    1, "dense_kernel");
    add_diag_kernel<<<(n + 255) / 256, 256, 0, c->st>>>(K.p, n, c->noise);
    c->check_launch(cudaGetLastError(), 1, "add_diag");
    int lwork = 0;
    CS(cusolverDnDpotrf_bufferSize(c->solver, CUBLAS_FILL_MODE_LOWER, n, K.p, n, &lwork));
    work.ensure(static_cast<size_t>(std::max(lwork, 1)));
    CS(cusolverDnDpotrf(c->solver, CUBLAS_FILL_MODE_LOWER, n, K.p, n, work.p, lwork, info.p));
    int hinfo = 0;
    c->d2h(&hinfo, info.p, sizeof(int));
    if (hinfo != 0) fail(GPK_NUMERICAL_ERROR, "mll_exact: Cholesky factorization failed; consider a larger noise variance");
    c->h2d(a.p, y, sizeof(double) * n);
    CS(cusolverDnDpotrs(c->solver, CUBLAS_FILL_MODE_LOWER, n, 1, K.p, n, a.p, n, info.p));
    std::vector<double> dg(n), ha(n);
    CK(cudaMemcpy2DAsync(dg.data(), sizeof(double), K.p, (static_cast<size_t>(n) + 1) * sizeof(double),
                         sizeof(double), n, cudaMemcpyDeviceToHost, c->st));
    c->d2h(ha.data(), a.p, sizeof(double) * n);
    double ld = 0.0, q = 0.0;
    for (int i = 0; i < n; ++i) ld += std::log(dg[i]);
    for (int i = 0; i < n; ++i) q += y[i] * ha[i];
    *value = -0.5 * (q + 2.0 * ld + static_cast<double>(n) * std::log(2.0 * 3.14159265358979323846));
    if (!gradient) return;
    // K_hat^{-1} (lower triangle) in place of the factor
    int lw2 = 0;
    CS(cusolverDnDpotri_bufferSize(c->solver, CUBLAS_FILL_MODE_LOWER, n, K.p, n, &lw2));
    work.ensure(static_cast<size_t>(std::max(lw2, 1)));
    CS(cusolverDnDpotri(c->solver, CUBLAS_FILL_MODE_LOWER, n, K.p, n, work.p, lw2, info.p));
    DBuf<double> dK, dka;
    dK.ensure(static_cast<size_t>(n) * n);
    dka.ensure(n);
    const double one = 1.0, zero = 0.0;
    std::vector<double> hp(n), hk(n);
    for (int w = 0; w < c->d + 2; ++w) {
      double quad = 0.0, tr = 0.0, raw = c->noise;
      if (w == c->d + 1) {  // dK_hat / dsigma^2 = I
        for (int i = 0; i < n; ++i) quad += ha[i] * ha[i];
        CK(cudaMemcpy2DAsync(hp.data(), sizeof(double), K.p, (static_cast<size_t>(n) + 1) * sizeof(double),
                             sizeof(double), n, cudaMemcpyDeviceToHost, c->st));
        c->sync();
        for (int i = 0; i < n; ++i) tr += hp[i];
      } else {
        double fac = 2.0 / c->o;  // kernel_deriv_column scale factors (kernels.hpp:252-267)
        raw = c->o;
        if (w >= 1) {
          const double lj = c->ls[w - 1];
          fac = -2.0 * c->o2 / (lj * lj * lj);
          raw = lj;
        }
        c->check_launch(gpk::launch_dense_kernel(c->family, c->sx.p, c->X.p, c->sq.p, n, c->d, w, c->o2, fac, dK.p,
                                                 n, c->st),
                        1, "dense_kernel");
        CB(cublasDsymv(c->blas, CUBLAS_FILL_MODE_LOWER, n, &one, dK.p, n, a.p, 1, &zero, dka.p, 1));
        c->check_launch(gpk::launch_sym_frob_partials(K.p, n, dK.p, n, n, part.p, c->st), 1, "sym_frob");
        CK(cudaMemcpyAsync(hk.data(), dka.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->st));
        c->d2h(hp.data(), part.p, sizeof(double) * n);
        for (int i = 0; i < n; ++i) quad += ha[i] * hk[i];
        for (int i = 0; i < n; ++i) tr += hp[i];
      }
      gradient[w] = 0.5 * (quad - tr) * raw;
    }
  });
}

// out = cross_kernel(A, X) v (kernels.hpp:339-354): A is na x d (test points), v has n entries.
static void cross_common(gpk_ctx* c, const double* A, int64_t na, int64_t lda, const double* dv, double* out) {
  const int d = c->d;
  require(na >= 1 && lda >= na, "cross_kernel: dimension mismatch");
  std::vector<double> sa(static_cast<size_t>(na) * d), qa(static_cast<size_t>(na), 0.0);
  for (int j = 0; j < d; ++j)
    for (int64_t i = 0; i < na; ++i) {
      const double v = A[j * lda + i];
      if (!std::isfinite(v)) fail(GPK_INPUT_ERROR, "cross_kernel: non-finite test inputs");
      sa[j * na + i] = v / c->ls[j];
    }
  for (int64_t i = 0; i < na; ++i)
    for (int j = 0; j < d; ++j) qa[i] += sa[j * na + i] * sa[j * na + i];
  DBuf<double> dsa, dqa, dout;
  dsa.ensure(sa.size());
  dqa.ensure(qa.size());
  dout.ensure(static_cast<size_t>(na));
  c->h2d(dsa.p, sa.data(), sizeof(double) * sa.size());
  c->h2d(dqa.p, qa.data(), sizeof(double) * qa.size());
  c->check_launch(gpk::launch_cross_mvm(c->family, dsa.p, dqa.p, static_cast<int>(na), c->sx.p, c->sq.p, c->n, d,
                                        c->o2, dv, dout.p, c->st),
                  1, "cross_mvm");
  c->d2h(out, dout.p, sizeof(double) * na);
}

gpk_status gpk_cross_kernel_mvm(gpk_ctx* ctx, const double* A, int64_t na, int64_t lda, const double* v,
                                double* out) {
  return guard(ctx, [&] {
    gpk_ctx* c = ctx;
    c->require_ready();
    require(c->world == 1, "cross_kernel: not available on a row-sharded context");
    for (int i = 0; i < c->n; ++i)
      if (!std::isfinite(v[i])) fail(GPK_INPUT_ERROR, "KernelOperator: non-finite entries in input vector");
    DBuf<double> dv;
    dv.ensure(c->n);
    c->h2d(dv.p, v, sizeof(double) * c->n);
    cross_common(c, A, na, lda, dv.p, out);
  });
}

// run_training_arm's predictive mean (experiments.hpp:403-414): alpha = pcg_solve(K_hat, y)
// with the attached preconditioner (one mBCG column, fp64-certified in the reduced-precision
// modes), then mean = cross_kernel(A, X) alpha.  iters: CG iterations of the solve (nullable).
gpk_status gpk_predict_mean(gpk_ctx* ctx, const double* y, const double* A, int64_t na, int64_t lda,
                            const gpk_cg_cfg* cfg, double* mean, int* iters) {
  return guard(ctx, [&] {
    gpk_ctx* c = ctx;
    c->require_ready();
    require(c->world == 1, "cross_kernel: not available on a row-sharded context");
    require(cfg != nullptr, "gpk_predict_mean: null config");
    require(c->pkind != 0, "gpkrylov_cuda: no preconditioner");
    require(cfg->max_iters >= 1, "CgConfig: max_iters must be >= 1");
    require(cfg->rel_tol > 0.0 && cfg->rel_tol < 1.0, "CgConfig: rel_tol must be in (0, 1)");
    require(cfg->precision >= GPK_PREC_FP64 && cfg->precision <= GPK_PREC_TF32X3, "CgConfig: unknown precision");
    for (int i = 0; i < c->n; ++i)
      if (!std::isfinite(y[i])) fail(GPK_INPUT_ERROR, "KernelOperator: non-finite entries in input vector");
    DBuf<double> db, dx;
    db.ensure(c->ldn);
    dx.ensure(c->ldn);
    c->h2d(db.p, y, sizeof(double) * c->n);
    const bool fp64 = cfg->precision == GPK_PREC_FP64;
    c->use_tc = cfg->precision == GPK_PREC_TF32X3;
    gpk_ctx::CgOut r;
    try {
      r = c->mbcg(db.p, c->ldn, 1, cfg->max_iters, cfg->rel_tol, fp64, dx.p, c->ldn, nullptr, nullptr, nullptr);
    } catch (const GpkError& e) {
      int col;
      fail(GPK_SOLVER_ERROR, strip_col(e.msg, &col));
    }
    if (!fp64 && cfg->refine > 0) {
      double mr;
      c->refine(db.p, c->ldn, 1, dx.p, c->ldn, r, cfg->max_iters, cfg->rel_tol, cfg->refine, &mr);
    }
    if (iters) *iters = r.iters[0];
    cross_common(c, A, na, lda, dx.p, mean);
  });
}

gpk_status gpk_data_shape(const gpk_ctx* ctx, int64_t* n, int* d) {
  if (!ctx || !ctx->have_data) return GPK_INPUT_ERROR;
  if (n) *n = ctx->n;
  if (d) *d = ctx->d;
  return GPK_OK;
}

void gpk_set_error_internal(gpk_ctx* ctx, const char* msg) {
  if (ctx) ctx->err = msg ? msg : "";
}

gpk_status gpk_make_probes(int64_t n, int count, uint64_t seed, double* out) {
  return guard(nullptr, [&] { make_probes_impl(n, count, seed, out); });
}

gpk_status gpk_make_probes_device(gpk_ctx* ctx, int64_t n, int count, uint64_t seed, double* d_out) {
  return guard(ctx, [&] {
    require(ctx != nullptr && d_out != nullptr, "make_probes: null context or output");
    require(n >= 1, "make_probes: n must be >= 1");
    require(count >= 1, "make_probes: need at least one probe");
    ctx->check_launch(gpk::launch_make_probes(n, count, seed, d_out, ctx->st), 1, "make_probes");
  });
}

uint64_t gpk_mix_seed(uint64_t seed, uint64_t salt) { return mix_seed_impl(seed, salt); }

}  // extern "C"
