// C ABI of the sm_100a DG acoustic hot path (see include/hybridwave_b200.h).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <utility>
#include <atomic>
#include <string>

#include "hw_kernels.cuh"
#include "hw_tet_mma.cuh"
#include "hw_dense_mma.cuh"

namespace hw {

static thread_local std::string g_err;
static int fail(const char* msg) {
  g_err = msg;
  return 1;
}

// kernel launches issued through this library (every launch site calls
// check_launch once; a CUDA-graph replay issues its captured launches
// without passing here)
static std::atomic<long long> g_launches{0};

static int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return 2;
  }
  return 0;
}

// Raise the dynamic shared-memory limit once per kernel instantiation (the
// call is not a stream operation; doing it once keeps launches capturable).
template <typename KernelT>
static int set_smem(KernelT kernel, size_t bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;   // (device, kernel): per-device attribute
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  const std::pair<int, const void*> key(dev, (const void*)kernel);
  if (done.count(key)) return 0;
  if (bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)bytes);
    if (e != cudaSuccess) {
      g_err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e);
      return 3;
    }
  }
  done.insert(key);
  return 0;
}

// HW_TET_KERNEL=scalar selects the scalar dense_kernel for the fp64 dense
// types (tet, wedge, pyramid) for A/B checks; default: the DMMA kernels
static bool tet_scalar() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("HW_TET_KERNEL");
    v = (s && !strcmp(s, "scalar")) ? 1 : 0;
  }
  return v == 1;
}

// Makes the mesh's device current for the duration of an ABI call and
// restores the caller's afterwards: the stream handle the caller passes may
// be a device's legacy default stream (0), and set_smem / side_streams key on
// the current device, so launching from another current device would run
// the kernels on the wrong GPU against the mesh's pointers.
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(const hw_mesh_t* M) {
    if (!M || M->device < 0) return;
    if (cudaGetDevice(&prev) != cudaSuccess) { ok = false; return; }
    if (prev != M->device && cudaSetDevice(M->device) != cudaSuccess) ok = false;
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

#define HW_DEVICE_GUARD(M)                                        \
  DeviceGuard device_guard_(M);                                   \
  if (!device_guard_.ok) return fail("cannot make the mesh's device current")

static void subset_of(const hw_subset_t* sub, int t, int64_t K, const int32_t** list,
                      int64_t* n) {
  *list = nullptr;
  *n = K;
  if (sub && sub->n[t] >= 0) {
    *list = sub->idx[t];
    *n = sub->n[t];
  }
}

template <int N, int T, typename R>
static int launch_dense(const hw_mesh_t& M, const hw_fields_t& Q, const Epi& E,
                        const int32_t* list, int64_t n, cudaStream_t st) {
  using L = Smem<N, T, R>;
  // non-affine wedges: cubature scratch (Naw) behind the layout
  constexpr size_t NAW_BYTES =
      (T == HW_WEDGE) ? 16 + sizeof(R) * (size_t)L::EPB * Naw<N>::CS : 0;
  static_assert(L::BYTES + NAW_BYTES <= 227 * 1024, "dense_kernel shared memory");
  const size_t bytes = L::BYTES + (M.t[T].op[8] != nullptr ? NAW_BYTES : 0);
  int rc;
  if ((rc = set_smem(dense_kernel<N, T, R>, L::BYTES + NAW_BYTES))) return rc;
  dense_kernel<N, T, R><<<(unsigned)((n + L::EPB - 1) / L::EPB), NT, bytes, st>>>(M, Q, E,
                                                                                  list, n);
  return check_launch("dense_kernel");
}

// Per-device side streams for running the element types' kernels
// concurrently within one stage (env HW_CONCURRENT=0 disables).  Fork/join
// through events, so the pattern is legal inside CUDA-graph capture.
struct SideStreams {
  cudaStream_t s[HW_NTYPES];
  cudaEvent_t fork_ev, join_ev[HW_NTYPES];
  int fork(cudaStream_t st0) {
    cudaError_t e = cudaEventRecord(fork_ev, st0);
    for (int i = 0; i < HW_NTYPES && e == cudaSuccess; ++i) e = cudaStreamWaitEvent(s[i], fork_ev, 0);
    if (e != cudaSuccess) return fail((std::string("side stream fork: ") + cudaGetErrorString(e)).c_str());
    return 0;
  }
  int join(cudaStream_t st0, int n) {
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < HW_NTYPES && e == cudaSuccess; ++i) {
      e = cudaEventRecord(join_ev[i], s[i]);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(st0, join_ev[i], 0);
    }
    (void)n;
    if (e != cudaSuccess) return fail((std::string("side stream join: ") + cudaGetErrorString(e)).c_str());
    return 0;
  }
};

static SideStreams* side_streams() {
  static const bool on = [] {
    const char* e = getenv("HW_CONCURRENT");
    return !(e && e[0] == '0');
  }();
  if (!on) return nullptr;
  static std::mutex mu;
  static SideStreams* per_dev[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!per_dev[dev]) {
    SideStreams* ss = new SideStreams;
    bool ok = cudaEventCreateWithFlags(&ss->fork_ev, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; i < HW_NTYPES && ok; ++i)
      ok = cudaStreamCreateWithFlags(&ss->s[i], cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&ss->join_ev[i], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) return nullptr;
    per_dev[dev] = ss;
  }
  return per_dev[dev];
}

// shared-memory floor per CTA (bytes, env HW_SMEM_FLOOR; tuning experiments:
// fewer resident CTAs leave more of the SM's L1 for the operator matrices)
static size_t smem_floor() {
  static const size_t v = [] {
    const char* e = getenv("HW_SMEM_FLOOR");
    return e ? (size_t)atol(e) : (size_t)0;
  }();
  return v;
}

template <int N, int T, typename R>
static int launch_dense_mma(const hw_mesh_t& M, const hw_fields_t& Q, const Epi& E,
                            const int32_t* list, int64_t n, cudaStream_t st) {
  using L = DMma<N, T, R>;
  // high orders (N >= 6): the DMMA kernel exceeds the CTA's thread / smem limits
  if constexpr (L::BYTES > 220 * 1024 || L::NTH > 1024) {
    return launch_dense<N, T, R>(M, Q, E, list, n, st);
  } else {
  int rc;
  const size_t bytes = L::BYTES > smem_floor() ? L::BYTES : smem_floor();
  const unsigned grid = (unsigned)((n + L::E - 1) / L::E);
  if constexpr (L::SPLIT) {   // only the launched layout is instantiated
    if ((rc = set_smem(dense_mma_kernel<N, T, R>, bytes))) return rc;
    dense_mma_kernel<N, T, R><<<grid, L::NTH, bytes, st>>>(M, Q, E, list, n);
  } else {
    if ((rc = set_smem(dense_mma_kernel_big<N, T, R>, bytes))) return rc;
    dense_mma_kernel_big<N, T, R><<<grid, L::NTH, bytes, st>>>(M, Q, E, list, n);
  }
  return check_launch("dense_mma_kernel");
  }
}

template <int N, int T, typename R>
static int launch_traces_t(const hw_mesh_t& M, const hw_fields_t& Q, const hw_fields_t& TR,
                           const int32_t* list, int64_t n, cudaStream_t st) {
  constexpr int NP = TT<N, T>::NP;
  constexpr int EPB = (NT / NP) > 0 ? (NT / NP) : 1;
  trace_kernel<N, T, R><<<(unsigned)((n + EPB - 1) / EPB), NT, 0, st>>>(M, Q, TR, list, n);
  return check_launch("trace_kernel");
}

// wedge / pyramid traces on DMMA (scalar kernel where the DMMA layout
// does not fit a block)
template <int N, int T, typename R>
static int launch_traces_mma(const hw_mesh_t& M, const hw_fields_t& Q, const hw_fields_t& TR,
                             const int32_t* list, int64_t n, cudaStream_t st) {
  using L = DMma<N, T, R>;
  if constexpr (L::NTH > 1024) {
    return launch_traces_t<N, T, R>(M, Q, TR, list, n, st);
  } else {
    constexpr size_t bytes = sizeof(R) * (L::E * (L::EQ + L::GEOS) + 2) + sizeof(int) * L::E;
    int rc;
    if ((rc = set_smem(trace_mma_kernel<N, T, R>, bytes))) return rc;
    trace_mma_kernel<N, T, R><<<(unsigned)((n + L::E - 1) / L::E), L::NTH, bytes, st>>>(
        M, Q, TR, list, n);
    return check_launch("trace_mma_kernel");
  }
}

// face traces of every publishing type (wedge, pyramid, GL hex) of q -> TR
template <int N, typename R>
static int launch_traces_all(const hw_mesh_t& M, const hw_fields_t& Q, const hw_fields_t& TR,
                             const hw_subset_t* sub, cudaStream_t st) {
  int rc = 0;
  for (int t = 0; t < HW_NTYPES; ++t) {
    const int64_t K = M.t[t].K;
    if (K <= 0) continue;
    const bool pub = t == HW_WEDGE || t == HW_PYRAMID || (t == HW_HEX && M.formulation == HW_GL);
    if (!pub) continue;
    if (!TR.p[t]) return fail("missing trace buffer for a publishing element type");
    const int32_t* list;
    int64_t n;
    subset_of(sub, t, K, &list, &n);
    if (n <= 0) continue;
    if (t == HW_HEX) rc = launch_traces_t<N, HW_HEX, R>(M, Q, TR, list, n, st);
    else if (t == HW_WEDGE)   // non-affine wedges (op[8]): per-point 1/sqrt(J), scalar kernel
      rc = M.t[HW_WEDGE].op[8] == nullptr ? launch_traces_mma<N, HW_WEDGE, R>(M, Q, TR, list, n, st)
                                          : launch_traces_t<N, HW_WEDGE, R>(M, Q, TR, list, n, st);
    else rc = launch_traces_mma<N, HW_PYRAMID, R>(M, Q, TR, list, n, st);
    if (rc) return rc;
  }
  return 0;
}

template <int N, typename R, bool SK, bool SEM>
static int launch_hex(const hw_mesh_t& M, const hw_fields_t& Q, const Epi& E,
                      const int32_t* list, int64_t n, unsigned grid, cudaStream_t st) {
  using L = Smem<N, HW_HEX, R, HW_HEX_NT>;
  int rc;
  if (E.mode == MODE_LSRK) {
    if ((rc = set_smem(hex_kernel<N, R, SK, SEM, true>, L::BYTES))) return rc;
    hex_kernel<N, R, SK, SEM, true><<<grid, HW_HEX_NT, L::BYTES, st>>>(M, Q, E, list, n);
  } else {
    if ((rc = set_smem(hex_kernel<N, R, SK, SEM, false>, L::BYTES))) return rc;
    hex_kernel<N, R, SK, SEM, false><<<grid, HW_HEX_NT, L::BYTES, st>>>(M, Q, E, list, n);
  }
  return 0;
}

template <int N, typename R>
static int launch_rhs_all(const hw_mesh_t& M, const hw_fields_t& Q, const Epi& E,
                          const hw_subset_t* sub, cudaStream_t st0) {
  int rc = 0;
  int active[HW_NTYPES], na = 0;
  // launch order on the side streams: measured best on the hybrid:38 N=3
  // step is pyramid, hex, wedge, tet (+3% over tet-first; 2 % over the type order)
  static int order[HW_NTYPES] = {HW_PYRAMID, HW_HEX, HW_WEDGE, HW_TET};
  static const bool order_env = [] {   // HW_TYPE_ORDER=3102 (tuning experiments)
    const char* e = getenv("HW_TYPE_ORDER");
    if (!e) return true;
    // accepted only as a permutation of 0..3: a repeated digit would launch
    // one type's update twice, concurrently, on the same rows
    int seen = 0;
    bool ok = strlen(e) == HW_NTYPES;
    for (int i = 0; ok && i < HW_NTYPES; ++i) {
      const int d = e[i] - '0';
      ok = d >= 0 && d < HW_NTYPES && !(seen & (1 << d));
      seen |= ok ? 1 << d : 0;
    }
    if (ok) {
      for (int i = 0; i < HW_NTYPES; ++i) order[i] = e[i] - '0';
    } else {
      fprintf(stderr, "hybridwave_b200: ignoring HW_TYPE_ORDER=%s (not a permutation of 0123)\n", e);
    }
    return true;
  }();
  (void)order_env;
  for (int o = 0; o < HW_NTYPES; ++o) {
    const int t = order[o];
    const int32_t* list;
    int64_t n = 0;
    if (M.t[t].K > 0) subset_of(sub, t, M.t[t].K, &list, &n);
    if (n > 0) active[na++] = t;
  }
  SideStreams* ss = na > 1 ? side_streams() : nullptr;
  if (ss && (rc = ss->fork(st0))) return rc;
  // every exit after a successful fork joins the side streams back into st0
  // (an unjoined fork would invalidate a CUDA-graph capture and leave st0
  // unordered after kernels already enqueued on the side streams)
  struct Joiner {
    SideStreams* ss;
    cudaStream_t st0;
    int na;
    ~Joiner() {
      if (ss) ss->join(st0, na);
    }
  };
  int join_rc = 0;
  {
  Joiner joiner{ss, st0, na};
  for (int a = 0; a < na; ++a) {
    const int t = active[a];
    const int64_t K = M.t[t].K;
    const int32_t* list;
    int64_t n;
    subset_of(sub, t, K, &list, &n);
    // the element types are independent within a stage: with side streams
    // their kernels run concurrently (fills the SMs past each kernel's tail)
    cudaStream_t st = ss ? ss->s[a] : st0;
    switch (t) {
      case HW_HEX: {
        using L = Smem<N, HW_HEX, R, HW_HEX_NT>;
        const unsigned grid = (unsigned)((n + L::EPB - 1) / L::EPB);
        const bool skew = M.t[HW_HEX].form == HW_FORM_SKEW, sem = M.formulation == HW_SEM;
        if (skew && sem) rc = launch_hex<N, R, true, true>(M, Q, E, list, n, grid, st);
        else if (skew) rc = launch_hex<N, R, true, false>(M, Q, E, list, n, grid, st);
        else if (sem) rc = launch_hex<N, R, false, true>(M, Q, E, list, n, grid, st);
        else rc = launch_hex<N, R, false, false>(M, Q, E, list, n, grid, st);
        if (rc) return rc;
        rc = check_launch("hex_kernel");
        break;
      }
      case HW_WEDGE:   // fp64 DMMA for both storage precisions; non-affine wedges (op[8]): scalar
        rc = (!tet_scalar() && M.t[HW_WEDGE].op[8] == nullptr)
                 ? launch_dense_mma<N, HW_WEDGE, R>(M, Q, E, list, n, st)
                 : launch_dense<N, HW_WEDGE, R>(M, Q, E, list, n, st);
        break;
      case HW_PYRAMID:   // non-affine pyramids present (op[8]): scalar kernel
        rc = (!tet_scalar() && M.t[HW_PYRAMID].op[8] == nullptr)
                 ? launch_dense_mma<N, HW_PYRAMID, R>(M, Q, E, list, n, st)
                 : launch_dense<N, HW_PYRAMID, R>(M, Q, E, list, n, st);
        break;
      case HW_TET:
        if (tet_scalar() && M.t[HW_TET].form == HW_FORM_SKEW)
          return fail("the scalar tet kernel implements the strong form only");
        if (!tet_scalar()) {   // fp64 DMMA for both storage precisions
          using L = TetMma<N, R>;
          const unsigned grid = (unsigned)((n + L::E - 1) / L::E);
          if (M.t[HW_TET].form == HW_FORM_SKEW) {
            if ((rc = set_smem(tet_mma_kernel<N, R, true>, L::BYTES))) return rc;
            tet_mma_kernel<N, R, true><<<grid, L::NTH, L::BYTES, st>>>(M, Q, E, list, n);
          } else {
            if ((rc = set_smem(tet_mma_kernel<N, R, false>, L::BYTES))) return rc;
            tet_mma_kernel<N, R, false><<<grid, L::NTH, L::BYTES, st>>>(M, Q, E, list, n);
          }
          rc = check_launch("tet_mma_kernel");
        } else {
          rc = launch_dense<N, HW_TET, R>(M, Q, E, list, n, st);
        }
        break;
    }
    if (rc) return rc;
  }
  joiner.ss = nullptr;                     // normal path: join explicitly, keep its status
  if (ss) join_rc = ss->join(st0, na);
  }
  return join_rc;
}

#ifndef HW_MAX_ORDER
#define HW_MAX_ORDER 7
#endif

template <typename R>
static int dispatch_rhs(const hw_mesh_t& M, const hw_fields_t& Q, const Epi& E,
                        const hw_subset_t* sub, cudaStream_t st) {
  switch (M.N) {
    case 1: return launch_rhs_all<1, R>(M, Q, E, sub, st);
    case 2: return launch_rhs_all<2, R>(M, Q, E, sub, st);
    case 3: return launch_rhs_all<3, R>(M, Q, E, sub, st);
    case 4: return launch_rhs_all<4, R>(M, Q, E, sub, st);
    case 5: return launch_rhs_all<5, R>(M, Q, E, sub, st);
#if HW_MAX_ORDER >= 6
    case 6: return launch_rhs_all<6, R>(M, Q, E, sub, st);
#endif
#if HW_MAX_ORDER >= 7
    case 7: return launch_rhs_all<7, R>(M, Q, E, sub, st);
#endif
    default: return fail("polynomial order not compiled into this library");
  }
}

template <typename R>
static int dispatch_traces(const hw_mesh_t& M, const hw_fields_t& Q, const hw_fields_t& TR,
                           const hw_subset_t* sub, cudaStream_t st) {
  switch (M.N) {
    case 1: return launch_traces_all<1, R>(M, Q, TR, sub, st);
    case 2: return launch_traces_all<2, R>(M, Q, TR, sub, st);
    case 3: return launch_traces_all<3, R>(M, Q, TR, sub, st);
    case 4: return launch_traces_all<4, R>(M, Q, TR, sub, st);
    case 5: return launch_traces_all<5, R>(M, Q, TR, sub, st);
#if HW_MAX_ORDER >= 6
    case 6: return launch_traces_all<6, R>(M, Q, TR, sub, st);
#endif
#if HW_MAX_ORDER >= 7
    case 7: return launch_traces_all<7, R>(M, Q, TR, sub, st);
#endif
    default: return fail("polynomial order not compiled into this library");
  }
}

static int run_traces(const hw_mesh_t* M, const hw_fields_t* Q, const hw_fields_t* TR,
                      const hw_subset_t* sub, void* stream) {
  if (!M || !Q || !TR) return fail("null mesh, fields or trace buffers");
  cudaStream_t st = (cudaStream_t)stream;
  if (M->dtype == HW_F64) return dispatch_traces<double>(*M, *Q, *TR, sub, st);
  if (M->dtype == HW_F32) return dispatch_traces<float>(*M, *Q, *TR, sub, st);
  return fail("unknown dtype");
}

static int run_rhs(const hw_mesh_t* M, const hw_fields_t* Q, const Epi& E,
                   const hw_subset_t* sub, void* stream) {
  if (!M || !Q) return fail("null mesh or fields");
  cudaStream_t st = (cudaStream_t)stream;
  if (M->dtype == HW_F64) return dispatch_rhs<double>(*M, *Q, E, sub, st);
  if (M->dtype == HW_F32) return dispatch_rhs<float>(*M, *Q, E, sub, st);
  return fail("unknown dtype");
}

// ---------------------------------------------------------------- elementwise

// out = q + dt (c0 h0 + c1 h1 + c2 h2) on the listed element rows (MRAB
// dense output); dt == 0 is a plain row copy (no history reads).  Element
// rows (4 Np scalars) are even-length: two scalars per thread.
// all element types in one launch (blockIdx.y = type): the multi-rate
// dense-output pass runs it on small per-level subsets, where per-type
// launches were latency-bound
struct Axpy3Types {
  const void* q[HW_NTYPES];
  void* out[HW_NTYPES];
  const void* h0[HW_NTYPES];
  const void* h1[HW_NTYPES];
  const void* h2[HW_NTYPES];
  const int32_t* list[HW_NTYPES];
  int64_t n[HW_NTYPES];
  int chunk[HW_NTYPES];
};

template <typename R>
__global__ void axpy3_kernel(Axpy3Types a, int nh, R c0, R c1, R c2, R dt) {
  const int t = blockIdx.y;
  const int64_t n = a.n[t];
  if (n <= 0) return;
  const R* __restrict__ q = (const R*)a.q[t];
  R* __restrict__ out = (R*)a.out[t];
  const R* __restrict__ h0 = (const R*)a.h0[t];
  const R* __restrict__ h1 = (const R*)a.h1[t];
  const R* __restrict__ h2 = (const R*)a.h2[t];
  const int32_t* __restrict__ list = a.list[t];
  const int chunk = a.chunk[t];
  const int half = chunk >> 1;
  const int64_t total = n * half;
  const bool copy = dt == R(0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = i / half;
    const int r = (int)(i - w * half);
    const size_t idx = (size_t)(list ? list[w] : w) * chunk + 2 * r;
    const R q0 = q[idx], q1 = q[idx + 1];
    if (copy) {
      out[idx] = q0;
      out[idx + 1] = q1;
      continue;
    }
    R a0 = c0 * h0[idx], a1 = c0 * h0[idx + 1];
    if (nh > 1) { a0 += c1 * h1[idx]; a1 += c1 * h1[idx + 1]; }
    if (nh > 2) { a0 += c2 * h2[idx]; a1 += c2 * h2[idx + 1]; }
    out[idx] = q0 + dt * a0;
    out[idx + 1] = q1 + dt * a1;
  }
}

template <typename R>
__global__ void hist_push_kernel(R* __restrict__ h0, R* __restrict__ h1, R* __restrict__ h2,
                                 const R* __restrict__ rhs, const int32_t* __restrict__ list,
                                 int64_t n, int chunk) {
  const int64_t total = n * chunk;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = i / chunk;
    const int r = (int)(i - w * chunk);
    const size_t idx = (size_t)(list ? list[w] : w) * chunk + r;
    h2[idx] = h1[idx];
    h1[idx] = h0[idx];
    h0[idx] = rhs[idx];
  }
}

template <typename R>
__global__ void pack_kernel(const R* __restrict__ q, const int32_t* __restrict__ idx, int64_t n,
                            int chunk, R* __restrict__ out) {
  const int64_t total = n * chunk;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = i / chunk;
    const int r = (int)(i - w * chunk);
    out[i] = q[(size_t)idx[w] * chunk + r];
  }
}

// Forcing residual of the pressure equation (hybridwave/dg.py:508-515 with
// the mass inverse of dg.py:479-490 and kappa): one thread per (element,
// node),
//   F[k][n] = kappa_k nodefac[k][n] sum_q B[n][q] f[k][q] scale[k][q],
// then out1[k][0][n] += alpha F, out2[k][0][n] += beta F (optional).
template <typename R>
__global__ void forcing_kernel(const double* __restrict__ f, const double* __restrict__ B,
                               const double* __restrict__ scale,
                               const double* __restrict__ nodefac, const R* __restrict__ mat,
                               int64_t K, int np, int nq, double alpha, R* __restrict__ out1,
                               double beta, R* __restrict__ out2, int assign) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K * np;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / np;
    const int n = (int)(i - k * np);
    const double* fk = f + k * nq;
    const double* sk = scale + k * nq;
    const double* b = B + (size_t)n * nq;
    double acc = 0.0;
    for (int qd = 0; qd < nq; ++qd) acc += b[qd] * (fk[qd] * sk[qd]);
    const double F = (double)mat[k * 4] * nodefac[i] * acc;
    const size_t o = (size_t)k * 4 * np + n;
    if (assign) {
      out1[o] = R(alpha * F);
    } else {
      out1[o] = R((double)out1[o] + alpha * F);
      if (out2) out2[o] = R((double)out2[o] + beta * F);
    }
  }
}

// Tet faces across a non-affine wedge's triangle (device.wedge_face_
// corrections): one block per (tet, face) pair adds the lift of the flux of
// delta = (L nb) * (s - 1) at the reference's face cubature points to the
// extra-RHS buffer `out` (state layout, all four fields).  nb: the wedge's
// published (unscaled) triangle trace at my face nodes.
template <typename R>
__global__ void wedge_face_corr_kernel(const R* __restrict__ trw, int nfp_w,
                                       const R* __restrict__ mat, double pen, int np, int nfn,
                                       int nq, const int* __restrict__ idata,
                                       const double* __restrict__ fdata,
                                       const double* __restrict__ Lall,
                                       const double* __restrict__ Pall, R* __restrict__ out) {
  extern __shared__ double wsm[];
  double* nb = wsm;                 // [4][nfn]
  double* dfp = nb + 4 * nfn;       // [nq]
  double* dfu = dfp + nq;           // [nq]
  const int* ir = idata + (size_t)blockIdx.x * (2 + nfn);
  const double* fr = fdata + (size_t)blockIdx.x * (6 + nq + np);
  const int k = ir[0], f = ir[1];
  for (int i = threadIdx.x; i < 4 * nfn; i += blockDim.x) {
    const int c = i / nfn, jj = i - c * nfn;
    nb[i] = (double)trw[(size_t)ir[2 + jj] + (size_t)c * nfp_w];
  }
  __syncthreads();
  const double tp = pen * fr[1], tu = pen * fr[0];
  const double n0 = fr[2], n1 = fr[3], n2 = fr[4], js = fr[5];
  const double* sm1 = fr + 6;
  const double* L = Lall + (size_t)f * nq * nfn;
  for (int i = threadIdx.x; i < nq; i += blockDim.x) {
    double d[4] = {0.0, 0.0, 0.0, 0.0};
    for (int jj = 0; jj < nfn; ++jj) {
      const double l = L[i * nfn + jj];
#pragma unroll
      for (int c = 0; c < 4; ++c) d[c] += l * nb[c * nfn + jj];
    }
    const double s = sm1[i];
    const double dp = d[0] * s, dun = (n0 * d[1] + n1 * d[2] + n2 * d[3]) * s;
    dfp[i] = 0.5 * tp * dp - 0.5 * dun;
    dfu[i] = 0.5 * tu * dun - 0.5 * dp;
  }
  __syncthreads();
  const double* P = Pall + (size_t)f * np * nq;
  const double kap = (double)mat[(size_t)k * 4], irho = (double)mat[(size_t)k * 4 + 1];
  for (int n = threadIdx.x; n < np; n += blockDim.x) {
    double sp = 0.0, su = 0.0;
    for (int i = 0; i < nq; ++i) {
      const double pv = P[n * nq + i];
      sp += pv * dfp[i];
      su += pv * dfu[i];
    }
    const double fac = js * fr[6 + nq + n];
    R* o = out + (size_t)k * 4 * np + n;
    atomicAdd(o, R(kap * fac * sp));
    atomicAdd(o + np, R(irho * fac * n0 * su));
    atomicAdd(o + 2 * np, R(irho * fac * n1 * su));
    atomicAdd(o + 3 * np, R(irho * fac * n2 * su));
  }
}

// face-level halo: buf[c * n + i] = src[off[i] + c * stride] (gather) and
// dst[off[i] + c * stride] = buf[c * n + i] (scatter), c = 0..3 fields
template <typename R>
__global__ void halo_gather_kernel(const R* __restrict__ src, int64_t stride,
                                   const int64_t* __restrict__ off, int64_t n,
                                   R* __restrict__ buf) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 4 * n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / n, j = i - c * n;
    buf[i] = src[off[j] + c * stride];
  }
}

template <typename R>
__global__ void halo_scatter_kernel(const R* __restrict__ buf, int64_t stride,
                                    const int64_t* __restrict__ off, int64_t n,
                                    R* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 4 * n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / n, j = i - c * n;
    dst[off[j] + c * stride] = buf[i];
  }
}

static int np_of(int t, int N) {
  switch (t) {
    case HW_HEX: return (N + 1) * (N + 1) * (N + 1);
    case HW_WEDGE: return (N + 1) * (N + 1) * (N + 2) / 2;
    case HW_PYRAMID: return (N + 1) * (N + 2) * (2 * N + 3) / 6;
    default: return (N + 1) * (N + 2) * (N + 3) / 6;
  }
}

static unsigned grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  return (unsigned)(g > 0 ? g : 1);
}

}  // namespace hw

using namespace hw;

// discrete energy per type (hw_energy)
template <int N, typename R>
static int launch_energy(const hw_mesh_t& M, const hw_fields_t& Q, double* out,
                         cudaStream_t st) {
  for (int t = 0; t < HW_NTYPES; ++t) {
    const int64_t K = M.t[t].K;
    if (K <= 0) continue;
    // one warp per element, 8 per block
    int64_t gb = (K + 7) / 8;
    if (gb > 148 * 16) gb = 148 * 16;
    const unsigned g = (unsigned)(gb > 0 ? gb : 1);
    switch (t) {
      case HW_HEX: energy_kernel<N, HW_HEX, R><<<g, 256, 0, st>>>(M, Q, out, K); break;
      case HW_WEDGE: energy_kernel<N, HW_WEDGE, R><<<g, 256, 0, st>>>(M, Q, out, K); break;
      case HW_PYRAMID: energy_kernel<N, HW_PYRAMID, R><<<g, 256, 0, st>>>(M, Q, out, K); break;
      default: energy_kernel<N, HW_TET, R><<<g, 256, 0, st>>>(M, Q, out, K); break;
    }
    int rc = check_launch("energy_kernel");
    if (rc) return rc;
  }
  return 0;
}

template <typename R>
static int dispatch_energy(const hw_mesh_t& M, const hw_fields_t& Q, double* out,
                           cudaStream_t st) {
  switch (M.N) {
    case 1: return launch_energy<1, R>(M, Q, out, st);
    case 2: return launch_energy<2, R>(M, Q, out, st);
    case 3: return launch_energy<3, R>(M, Q, out, st);
    case 4: return launch_energy<4, R>(M, Q, out, st);
    case 5: return launch_energy<5, R>(M, Q, out, st);
#if HW_MAX_ORDER >= 6
    case 6: return launch_energy<6, R>(M, Q, out, st);
#endif
#if HW_MAX_ORDER >= 7
    case 7: return launch_energy<7, R>(M, Q, out, st);
#endif
    default: return fail("polynomial order not compiled into this library");
  }
}

extern "C" {

int hw_version(void) { return 1; }

long long hw_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int hw_supported_orders(void) {
  int m = 0;
  for (int n = 1; n <= HW_MAX_ORDER; ++n) m |= 1 << n;
  return m;
}

const char* hw_last_error(void) { return g_err.c_str(); }

int hw_traces(const hw_mesh_t* mesh, const hw_fields_t* q, hw_fields_t* tr,
              const hw_subset_t* subset, void* stream) {
  HW_DEVICE_GUARD(mesh);
  return run_traces(mesh, q, tr, subset, stream);
}

int hw_rhs(const hw_mesh_t* mesh, const hw_fields_t* q, hw_fields_t* rhs,
           const hw_subset_t* subset, void* stream) {
  HW_DEVICE_GUARD(mesh);
  if (!rhs) return fail("null rhs");
  if (!mesh) return fail("null mesh");
  {   // traces of q for the publishing types, on every element (neighbours of
      // a subset need them too)
    hw_fields_t tr;
    for (int t = 0; t < HW_NTYPES; ++t) tr.p[t] = mesh->tr_in[t];
    int rc = run_traces(mesh, q, &tr, nullptr, stream);
    if (rc) return rc;
  }
  Epi E;
  memset(&E, 0, sizeof(E));
  for (int t = 0; t < HW_NTYPES; ++t) E.frc[t] = mesh->frc[t];
  E.mode = MODE_RHS;
  for (int t = 0; t < HW_NTYPES; ++t) E.out[t] = rhs->p[t];
  return run_rhs(mesh, q, E, subset, stream);
}

int hw_lsrk_stage(const hw_mesh_t* mesh, const hw_fields_t* q_in, hw_fields_t* q_out,
                  hw_fields_t* res, double a, double b, double dt, const hw_subset_t* subset,
                  void* stream) {
  HW_DEVICE_GUARD(mesh);
  if (!q_out || !res) return fail("null q_out/res");
  Epi E;
  memset(&E, 0, sizeof(E));
  for (int t = 0; t < HW_NTYPES; ++t) E.frc[t] = mesh->frc[t];
  E.mode = MODE_LSRK;
  E.a = a;
  E.b = b;
  E.dt = dt;
  for (int t = 0; t < HW_NTYPES; ++t) {
    if (mesh->t[t].K > 0 && q_in->p[t] == q_out->p[t]) return fail("q_in and q_out must differ");
    E.res[t] = res->p[t];
    E.qout[t] = q_out->p[t];
  }
  return run_rhs(mesh, q_in, E, subset, stream);
}

int hw_ab_step(const hw_mesh_t* mesh, const hw_fields_t* q_in, hw_fields_t* q_out,
               hw_fields_t* h0, const hw_fields_t* h1, const hw_fields_t* h2, int n_hist,
               double c0, double c1, double c2, double dt, const hw_subset_t* subset,
               void* stream) {
  HW_DEVICE_GUARD(mesh);
  if (n_hist < 1 || n_hist > 3) return fail("history depth must be 1..3");
  Epi E;
  memset(&E, 0, sizeof(E));
  for (int t = 0; t < HW_NTYPES; ++t) E.frc[t] = mesh->frc[t];
  E.mode = MODE_AB;
  E.nhist = n_hist;
  E.c0 = c0;
  E.c1 = c1;
  E.c2 = c2;
  E.dt = dt;
  for (int t = 0; t < HW_NTYPES; ++t) {
    if (mesh->t[t].K > 0 && q_in->p[t] == q_out->p[t]) return fail("q_in and q_out must differ");
    E.out[t] = h0->p[t];
    E.qout[t] = q_out->p[t];
    E.h1[t] = h1 ? h1->p[t] : nullptr;
    E.h2[t] = h2 ? h2->p[t] : nullptr;
  }
  return run_rhs(mesh, q_in, E, subset, stream);
}

int hw_axpy3(const hw_mesh_t* mesh, const hw_fields_t* q, hw_fields_t* out,
             const hw_fields_t* h0, const hw_fields_t* h1, const hw_fields_t* h2, int n_hist,
             double c0, double c1, double c2, double dt, const hw_subset_t* subset,
             void* stream) {
  HW_DEVICE_GUARD(mesh);
  cudaStream_t st = (cudaStream_t)stream;
  Axpy3Types a{};
  unsigned g = 0;
  for (int t = 0; t < HW_NTYPES; ++t) {
    const int64_t K = mesh->t[t].K;
    a.n[t] = 0;
    if (K <= 0) continue;
    subset_of(subset, t, K, &a.list[t], &a.n[t]);
    if (a.n[t] <= 0) continue;
    a.chunk[t] = 4 * np_of(t, mesh->N);
    a.q[t] = q->p[t];
    a.out[t] = out->p[t];
    a.h0[t] = h0->p[t];
    a.h1[t] = h1 ? h1->p[t] : nullptr;
    a.h2[t] = h2 ? h2->p[t] : nullptr;
    const unsigned gt = grid_for(a.n[t] * a.chunk[t] / 2);
    g = gt > g ? gt : g;
  }
  if (g == 0) return 0;
  const dim3 grid(g, HW_NTYPES);
  if (mesh->dtype == HW_F64)
    axpy3_kernel<double><<<grid, 256, 0, st>>>(a, n_hist, c0, c1, c2, dt);
  else
    axpy3_kernel<float><<<grid, 256, 0, st>>>(a, n_hist, (float)c0, (float)c1, (float)c2,
                                              (float)dt);
  return check_launch("axpy3_kernel");
}

int hw_hist_push(const hw_mesh_t* mesh, hw_fields_t* h0, hw_fields_t* h1, hw_fields_t* h2,
                 const hw_fields_t* rhs, const hw_subset_t* subset, void* stream) {
  HW_DEVICE_GUARD(mesh);
  cudaStream_t st = (cudaStream_t)stream;
  for (int t = 0; t < HW_NTYPES; ++t) {
    const int64_t K = mesh->t[t].K;
    if (K <= 0) continue;
    const int32_t* list;
    int64_t n;
    subset_of(subset, t, K, &list, &n);
    if (n <= 0) continue;
    const int chunk = 4 * np_of(t, mesh->N);
    const unsigned g = grid_for(n * chunk);
    if (mesh->dtype == HW_F64)
      hist_push_kernel<double><<<g, 256, 0, st>>>((double*)h0->p[t], (double*)h1->p[t],
                                                  (double*)h2->p[t], (const double*)rhs->p[t],
                                                  list, n, chunk);
    else
      hist_push_kernel<float><<<g, 256, 0, st>>>((float*)h0->p[t], (float*)h1->p[t],
                                                 (float*)h2->p[t], (const float*)rhs->p[t], list,
                                                 n, chunk);
    int rc = check_launch("hist_push_kernel");
    if (rc) return rc;
  }
  return 0;
}

int hw_halo_pack(const hw_mesh_t* mesh, int elem_type, const void* q, const int32_t* idx,
                 int64_t n, void* sendbuf, void* stream) {
  HW_DEVICE_GUARD(mesh);
  if (elem_type < 0 || elem_type >= HW_NTYPES) return fail("bad element type");
  if (n <= 0) return 0;
  const int chunk = 4 * np_of(elem_type, mesh->N);
  const unsigned g = grid_for(n * chunk);
  cudaStream_t st = (cudaStream_t)stream;
  if (mesh->dtype == HW_F64)
    pack_kernel<double><<<g, 256, 0, st>>>((const double*)q, idx, n, chunk, (double*)sendbuf);
  else
    pack_kernel<float><<<g, 256, 0, st>>>((const float*)q, idx, n, chunk, (float*)sendbuf);
  return check_launch("pack_kernel");
}

int hw_halo_gather(const hw_mesh_t* mesh, const void* src, int64_t stride, const int64_t* off,
                   int64_t n, void* buf, void* stream) {
  HW_DEVICE_GUARD(mesh);
  if (n <= 0) return 0;
  if (!src || !off || !buf) return fail("hw_halo_gather: null pointer");
  const unsigned g = grid_for(4 * n);
  cudaStream_t st = (cudaStream_t)stream;
  if (mesh->dtype == HW_F64)
    halo_gather_kernel<double><<<g, 256, 0, st>>>((const double*)src, stride, off, n,
                                                  (double*)buf);
  else
    halo_gather_kernel<float><<<g, 256, 0, st>>>((const float*)src, stride, off, n,
                                                 (float*)buf);
  return check_launch("halo_gather_kernel");
}

int hw_halo_scatter(const hw_mesh_t* mesh, const void* buf, int64_t stride, const int64_t* off,
                    int64_t n, void* dst, void* stream) {
  HW_DEVICE_GUARD(mesh);
  if (n <= 0) return 0;
  if (!dst || !off || !buf) return fail("hw_halo_scatter: null pointer");
  const unsigned g = grid_for(4 * n);
  cudaStream_t st = (cudaStream_t)stream;
  if (mesh->dtype == HW_F64)
    halo_scatter_kernel<double><<<g, 256, 0, st>>>((const double*)buf, stride, off, n,
                                                   (double*)dst);
  else
    halo_scatter_kernel<float><<<g, 256, 0, st>>>((const float*)buf, stride, off, n,
                                                  (float*)dst);
  return check_launch("halo_scatter_kernel");
}

int hw_forcing(const hw_mesh_t* mesh, int elem_type, const double* f, const double* B,
               const double* scale, const double* nodefac, int nq, double alpha, void* out1,
               double beta, void* out2, int assign, void* stream) {
  HW_DEVICE_GUARD(mesh);
  if (elem_type < 0 || elem_type >= HW_NTYPES) return fail("bad element type");
  const int64_t K = mesh->t[elem_type].K;
  if (K <= 0) return 0;
  if (!f || !B || !scale || !nodefac || !out1 || nq <= 0) return fail("hw_forcing: bad arguments");
  const int np = np_of(elem_type, mesh->N);
  const unsigned g = grid_for(K * np);
  cudaStream_t st = (cudaStream_t)stream;
  if (mesh->dtype == HW_F64)
    forcing_kernel<double><<<g, 256, 0, st>>>(f, B, scale, nodefac,
                                              (const double*)mesh->t[elem_type].mat, K, np, nq,
                                              alpha, (double*)out1, beta, (double*)out2,
                                              assign);
  else
    forcing_kernel<float><<<g, 256, 0, st>>>(f, B, scale, nodefac,
                                             (const float*)mesh->t[elem_type].mat, K, np, nq,
                                             alpha, (float*)out1, beta, (float*)out2,
                                             assign);
  return check_launch("forcing_kernel");
}

int hw_wedge_face_correction(const hw_mesh_t* mesh, int elem_type, int n_pairs,
                             const int32_t* idata, const double* fdata, const double* L,
                             const double* P, int nq, int nfn, void* out, void* stream) {
  HW_DEVICE_GUARD(mesh);
  if (n_pairs <= 0) return 0;
  if (elem_type != HW_TET && elem_type != HW_PYRAMID)
    return fail("hw_wedge_face_correction: tets and pyramids only");
  if (!mesh->tr_in[HW_WEDGE]) return fail("hw_wedge_face_correction: no wedge traces");
  const int np = np_of(elem_type, mesh->N), nfp_w = [&] {
    const int N = mesh->N, nfn_ = (N + 1) * (N + 2) / 2, nfq = (N + 1) * (N + 1);
    return 2 * nfn_ + 3 * nfq;
  }();
  const size_t smem = sizeof(double) * (4 * nfn + 2 * nq);
  cudaStream_t st = (cudaStream_t)stream;
  if (mesh->dtype == HW_F64)
    wedge_face_corr_kernel<double><<<n_pairs, 128, smem, st>>>(
        (const double*)mesh->tr_in[HW_WEDGE], nfp_w, (const double*)mesh->t[elem_type].mat,
        mesh->penalty_scale, np, nfn, nq, idata, fdata, L, P, (double*)out);
  else
    wedge_face_corr_kernel<float><<<n_pairs, 128, smem, st>>>(
        (const float*)mesh->tr_in[HW_WEDGE], nfp_w, (const float*)mesh->t[elem_type].mat,
        mesh->penalty_scale, np, nfn, nq, idata, fdata, L, P, (float*)out);
  return check_launch("wedge_face_corr_kernel");
}

int hw_prepare(const hw_mesh_t* mesh) {
  HW_DEVICE_GUARD(mesh);
  if (!mesh) return fail("null mesh");
  if (mesh->N < 1 || mesh->N > 7) return fail("polynomial order out of range");
  if (mesh->t[HW_HEX].K > 0) {
    if (!mesh->t[HW_HEX].iop[3]) return fail("hex face-point table missing");
    const size_t off = sizeof(int) * 24 * ((size_t)mesh->formulation * 8 + mesh->N);
    cudaError_t e = cudaMemcpyToSymbol(c_hex_spc, mesh->t[HW_HEX].iop[3], 24 * sizeof(int),
                                       off, cudaMemcpyDeviceToDevice);
    if (e != cudaSuccess) return fail(cudaGetErrorString(e));
  }
  return 0;
}

int hw_energy(const hw_mesh_t* mesh, const hw_fields_t* q, double* out, void* stream) {
  HW_DEVICE_GUARD(mesh);
  if (!out) return fail("hw_energy: out is null");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(out, 0, HW_NTYPES * sizeof(double), st);
  if (e != cudaSuccess) return fail(cudaGetErrorString(e));
  return mesh->dtype == HW_F64 ? dispatch_energy<double>(*mesh, *q, out, st)
                               : dispatch_energy<float>(*mesh, *q, out, st);
}

}  // extern "C"
