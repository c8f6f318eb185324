// Fused per-element-type RHS + time-update kernels (sm_100a): the hex
// kernel, the scalar dense kernel (high-N / debug fallback for wedge,
// pyramid, tet), the hw_traces and hw_energy kernels, and the shared
// traits, copy helpers and epilogues (the DMMA tet / wedge / pyramid
// kernels are in hw_tet_mma.cuh / hw_dense_mma.cuh).
//
// One launch per element type per stage.  A block owns EPB elements:
//   P0 load       q rows, geometry records, materials, links (cp.async) and
//                 every face point's neighbour value through the host gather
//                 index (cp.async for hex, registers for the DMMA kernels),
//                 the LSRK residual behind the volume / lift work
//   P1 volume     strong/skew volume term, mass inverse folded out
//   P2 flux       own + neighbour traces, upwind flux x face Jacobian
//   P3 lift       face-to-volume lift, mass inverse, materials, epilogue
//                 (RHS / LSRK stage / AB step), publish the new traces
// Reference data flow: hybridwave/dg.py:299-506.
#pragma once
#include "hw_common.cuh"

namespace hw {

__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }

// ------------------------------------------------------------------ traits

template <int N, int T>
struct TT;

template <int N>
struct TT<N, HW_TET> {
  using D = Dims<N>;
  static constexpr int NP = D::NP_TET, NF = 4, NFP = D::NFP_TET, GEO = GEO_TET, GF = 9;
  __host__ __device__ static constexpr bool tri(int) { return true; }
  __host__ __device__ static constexpr int off(int f) { return f * D::NFN; }
  __host__ __device__ static constexpr int cnt(int) { return D::NFN; }
  __host__ __device__ static constexpr int stage(int) { return 4 * D::NFN; }
};

template <int N>
struct TT<N, HW_WEDGE> {
  using D = Dims<N>;
  static constexpr int NP = D::NP_WEDGE, NF = 5, NFP = D::NFP_WEDGE, GEO = GEO_WEDGE, GF = 10;
  __host__ __device__ static constexpr bool tri(int f) { return f < 2; }
  __host__ __device__ static constexpr int off(int f) {
    return f < 2 ? f * D::NFN : 2 * D::NFN + (f - 2) * D::NFQ;
  }
  __host__ __device__ static constexpr int cnt(int f) { return f < 2 ? D::NFN : D::NFQ; }
  __host__ __device__ static constexpr int stage(int f) { return 4 * cnt(f); }
};

// Non-affine LSC-DG wedges (op[8] present: every wedge of the mesh runs the
// scalar dense kernel).  The reference's two cubature passes with G and
// grad J at every volume cubature point (hybridwave/dg.py:423-444) and, on
// the triangle faces, its face cubature (dg.py:300-357): own and neighbour
// traces are published / staged as their polynomial part at the nodal face
// points, interpolated to the cubature points (exact: degree N) and scaled
// by each side's 1/sqrt(J) there.  Quad faces keep the device points (the
// reference's quad cubature) with per-point n, Js, 1/sqrt(J).
//   op[8] (K, GW): [NQ][12] w G[c][x], w gJfac[x] | [NFP][5] n, Js/sqrt(J),
//                  1/sqrt(J) (quad points) | [2][NQT][3] 1/sqrt(J) own,
//                  1/sqrt(J) neighbour, w Js/sqrt(J) (triangle cubature)
//   op[9]: V, Dr3, Ds3, Dt3 as [m][q] | the same as [q][m] | Lq [2][NQT][NFN]
//          | Vf [2][NQT][NP] (triangle faces)
template <int N>
struct Naw {
  using D = Dims<N>;
  // NQT: the reference's triangle face rule without its duplicate points
  // (6(N+1)^2 stored, each twice with equal weights: device.wedge_cubature_ops)
  static constexpr int NP = D::NP_WEDGE, NQ = D::NQ_WEDGE, NQT = 3 * D::N1 * D::N1,
                       NFN = D::NFN, NFP = D::NFP_WEDGE;
  static constexpr int GF = NQ * 12, GT = GF + NFP * 5, GW = GT + 2 * NQT * 3;
  static constexpr int CVN = 4 * NP * NQ, CLQ = 8 * NP * NQ, CVF = CLQ + 2 * NQT * NFN;
  // smem scratch per element: the trial-pass values, then (after the test
  // pass) the triangle-face fluxes
  static constexpr int CS = (7 * NQ > 4 * NQT) ? 7 * NQ : 4 * NQT;
};

template <int N>
struct TT<N, HW_PYRAMID> {
  using D = Dims<N>;
  static constexpr int NP = D::NP_PYR, NF = 5, NFP = D::NFP_PYR, GEO = GEO_PYR, GF = 9;
  __host__ __device__ static constexpr bool tri(int f) { return f > 0; }
  __host__ __device__ static constexpr int off(int f) {
    return f == 0 ? 0 : D::NFQ + (f - 1) * D::NFN;
  }
  __host__ __device__ static constexpr int cnt(int f) { return f == 0 ? D::NFQ : D::NFN; }
  __host__ __device__ static constexpr int stage(int f) { return 4 * cnt(f); }
};

template <int N>
struct TT<N, HW_HEX> {
  using D = Dims<N>;
  static constexpr int NP = D::NP_HEX, NF = 6, NFP = D::NFP_HEX, GEO = GEO_HEX, GF = 0;
  __host__ __device__ static constexpr bool tri(int) { return false; }
  __host__ __device__ static constexpr int off(int f) { return f * D::NFQ; }
  __host__ __device__ static constexpr int cnt(int) { return D::NFQ; }
  __host__ __device__ static constexpr int stage(int) { return 4 * D::NFQ; }
};

template <int N, int T>
__host__ __device__ constexpr int stage_off(int f) {
  int s = 0;
  for (int g = 0; g < TT<N, T>::NF; ++g) s += (g < f) ? TT<N, T>::stage(g) : 0;
  return s;
}

template <int N, int T>
__device__ __forceinline__ int face_of_point(int j, int& jj) {
  using X = TT<N, T>;
  int f = 0;
#pragma unroll
  for (int g = 1; g < X::NF; ++g)
    if (j >= X::off(g)) f = g;
  jj = j - X::off(f);
  return f;
}

// ------------------------------------------------------------------ cp.async

template <typename R>
__device__ __forceinline__ void cp_async(R* smem, const R* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  if (sizeof(R) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

// ne (<= EMAX) element rows of W scalars (W * sizeof(R) a multiple of 16),
// element k of the block at src + sk[k] * W, into dst + k * DW; 16 bytes
// per copy, loop fully unrolled over the compile-time trip count
template <int W, int DW, int NTHR, int EMAX, typename R>
__device__ __forceinline__ void copy_rows16(R* dst, const R* src, const int* sk, int ne) {
  constexpr int V = 16 / sizeof(R), CH = W / V, TOT = EMAX * CH;
#pragma unroll
  for (int u = 0; u < (TOT + NTHR - 1) / NTHR; ++u) {
    const int i = (int)threadIdx.x + u * NTHR;
    if ((TOT % NTHR) && i >= TOT) break;
    const int e = i / CH, c = i - e * CH;
    if (e >= ne) break;
    cp_async16(dst + e * DW + c * V, src + (size_t)sk[e] * W + c * V);
  }
}

// warp-per-element variants: warp w copies the rows of elements w, w + NW,
// ...; sk and the row bases are warp-uniform, one add per copy remains
template <int W, int DW, int NW, typename R>
__device__ __forceinline__ void copy_rows16_w(R* dst, const R* src, const int* sk, int ne) {
  constexpr int V = 16 / sizeof(R), CH = W / V;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int e = warp; e < ne; e += NW) {
    const R* s = src + (size_t)sk[e] * W;
    R* d = dst + e * DW;
#pragma unroll
    for (int c0 = 0; c0 < CH; c0 += 32)
      if (c0 + lane < CH) cp_async16(d + (c0 + lane) * V, s + (c0 + lane) * V);
  }
}

template <int W, int DW, int NW, typename R>
__device__ __forceinline__ void copy_rows_w(R* dst, const R* src, const int* sk, int ne) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int e = warp; e < ne; e += NW) {
    const R* s = src + (size_t)sk[e] * W;
    R* d = dst + e * DW;
#pragma unroll
    for (int c0 = 0; c0 < W; c0 += 32)
      if (c0 + lane < W) cp_async(d + c0 + lane, s + c0 + lane);
  }
}

// the same with one scalar per copy (rows of odd length, e.g. records)
template <int W, int DW, int NTHR, int EMAX, typename R>
__device__ __forceinline__ void copy_rows(R* dst, const R* src, const int* sk, int ne) {
  constexpr int TOT = EMAX * W;
#pragma unroll
  for (int u = 0; u < (TOT + NTHR - 1) / NTHR; ++u) {
    const int i = (int)threadIdx.x + u * NTHR;
    if ((TOT % NTHR) && i >= TOT) break;
    const int e = i / W, c = i - e * W;
    if (e >= ne) break;
    cp_async(dst + e * DW + c, src + (size_t)sk[e] * W + c);
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// Types whose face traces are published in the trace buffers (their traces
// are dense contractions / interpolations); tets and SEM hexes are read
// straight from the state (their traces are selections).
__device__ __forceinline__ bool publishes(int t, bool sem) {
  return t == HW_WEDGE || t == HW_PYRAMID || (t == HW_HEX && !sem);
}

template <int N>
__device__ __forceinline__ int nfp_of(int t) {
  using D = Dims<N>;
  return t == HW_HEX ? D::NFP_HEX : t == HW_TET ? D::NFP_TET
                     : t == HW_WEDGE ? D::NFP_WEDGE : D::NFP_PYR;
}

// P1: one warp per (element, face) pair copies the neighbour's face values
// (4 fields x cnt points, in the neighbour's own point order): a contiguous
// trace-buffer row for publishing neighbours, selected face nodes of the
// state for tets and SEM hexes.
template <int N, int T, typename R>
__device__ __forceinline__ void stage_neighbours(const hw_mesh_t& M, const hw_fields_t& Q,
                                                 const int* snc, const int* sne, int ne,
                                                 R* st, bool sem) {
  using X = TT<N, T>;
  using D = Dims<N>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int pr = warp; pr < ne * X::NF; pr += NT / 32) {
    const int e = pr / X::NF, f = pr - e * X::NF;
    const int code = snc[pr];
    if (code & HW_NBR_BOUNDARY) continue;
    const int t2 = HW_NBR_TYPE(code), f2 = HW_NBR_FACE(code);
    const int k2 = sne[pr];
    const int cnt = X::cnt(f);
    R* dst = st + e * stage_off<N, T>(X::NF) + stage_off<N, T>(f);
    if (publishes(t2, sem)) {
      const int nfp2 = nfp_of<N>(t2);
      const R* src = (const R*)M.tr_in[t2] + (size_t)k2 * 4 * nfp2 + face_offset<N>(t2, f2);
      for (int i = lane; i < 4 * cnt; i += 32) {
        const int c = i / cnt, p = i - c * cnt;
        cp_async(dst + i, src + c * nfp2 + p);
      }
    } else if (t2 == HW_TET) {
      const R* q2 = (const R*)Q.p[HW_TET] + (size_t)k2 * 4 * D::NP_TET;
      const int* fn = M.t[HW_TET].iop[0] + f2 * D::NFN;
      for (int i = lane; i < 4 * D::NFN; i += 32) {
        const int c = i / D::NFN, n = i - c * D::NFN;
        cp_async(dst + i, q2 + c * D::NP_TET + __ldg(fn + n));
      }
    } else {   // SEM hex: face nodes
      const R* q2 = (const R*)Q.p[HW_HEX] + (size_t)k2 * 4 * D::NP_HEX;
      const int* tab = M.t[HW_HEX].iop[0] + 3 * f2 * D::NFQ;
      for (int i = lane; i < 4 * D::NFQ; i += 32) {
        const int c = i / D::NFQ, p = i - c * D::NFQ;
        const int base = __ldg(tab + 3 * p), stride = __ldg(tab + 3 * p + 1),
                  end = __ldg(tab + 3 * p + 2);
        cp_async(dst + i, q2 + c * D::NP_HEX + base + (end ? N : 0) * stride);
      }
    }
  }
}

// neighbour trace at my face point jj from the staged face values
template <int N, int T, typename R>
__device__ __forceinline__ void staged_trace(const hw_mesh_t& M, int code, int f, int jj,
                                             const R* st_e, R tr[4]) {
  using X = TT<N, T>;
  using D = Dims<N>;
  const int pc = HW_NBR_PERM(code);
  const int cnt = X::cnt(f);
  const int p = X::tri(f) ? __ldg(M.perm_tri + pc * D::NFN + jj)
                          : __ldg(M.perm_quad + pc * D::NFQ + jj);
  const R* s = st_e + stage_off<N, T>(f);
#pragma unroll
  for (int c = 0; c < 4; ++c) tr[c] = s[c * cnt + p];
}

// Face traces of element states held element-major in smem (sq[e][c][n],
// element stride 4*Np) -> trace buffer rows tr[k][c][j].  Dense types:
// E q (wedge x 1/sqrt(J)); GL hex: 1-D endpoint interpolation.
template <int N, int T, typename R>
__device__ __forceinline__ void publish_traces(const hw_mesh_t& M, const R* sq, const R* sg,
                                               const int* sk, int ne, R* tr) {
  using X = TT<N, T>;
  using D = Dims<N>;
  constexpr int NP = X::NP, NFP = X::NFP;
  const hw_type_t& TY = M.t[T];
  for (int i = threadIdx.x; i < ne * NFP; i += blockDim.x) {
    const int e = i / NFP, j = i - e * NFP;
    const R* qe = sq + e * 4 * NP;
    R a0 = R(0), a1 = R(0), a2 = R(0), a3 = R(0);
    if (T == HW_HEX) {
      const int* tab = TY.iop[0] + 3 * j;
      const int base = __ldg(tab), stride = __ldg(tab + 1), end = __ldg(tab + 2);
      const R* ve = (const R*)TY.op[1] + end * D::N1;
#pragma unroll
      for (int l = 0; l < D::N1; ++l) {
        const R w = ldg(ve + l);
        const int n = base + l * stride;
        a0 += w * qe[n]; a1 += w * qe[NP + n]; a2 += w * qe[2 * NP + n]; a3 += w * qe[3 * NP + n];
      }
    } else {
      const R* ET = (const R*)TY.op[5];
#pragma unroll 4
      for (int m = 0; m < NP; ++m) {
        const R ev = ldg(ET + m * NFP + j);
        a0 += ev * qe[m]; a1 += ev * qe[NP + m]; a2 += ev * qe[2 * NP + m]; a3 += ev * qe[3 * NP + m];
      }
      if (T == HW_WEDGE) {
        R isj = sg[e * X::GEO + 9];
        if (TY.op[8] != nullptr)   // non-affine: quad points x 1/sqrt(J), triangles polynomial
          isj = j < 2 * D::NFN ? R(1)
                               : ldg((const R*)TY.op[8] + (size_t)sk[e] * Naw<N>::GW +
                                     Naw<N>::GF + j * 5 + 4);
        a0 *= isj; a1 *= isj; a2 *= isj; a3 *= isj;
      }
    }
    R* o = tr + (size_t)sk[e] * 4 * NFP + j;
    o[0] = a0; o[NFP] = a1; o[2 * NFP] = a2; o[3 * NFP] = a3;
  }
}

// ------------------------------------------------------------------ smem layout

template <int N, int T, typename R, int NTH = NT>
struct Smem {
  using X = TT<N, T>;
  static constexpr int NP = X::NP, NF = X::NF, NFP = X::NFP;
  static constexpr int EPB = (NTH / NP) > 0 ? (NTH / NP) : 1;
  static constexpr int S = (EPB * NP + NTH - 1) / NTH;
  static constexpr int FLUXW = (T == HW_HEX) ? 4 : 2;       // flux words per face point
  static constexpr int STG = stage_off<N, T>(NF);           // staged values per element
  // rows copied with 16-byte cp.async first (even sizes keep them aligned)
  static constexpr int SQ = 0;
  static constexpr int SRES = SQ + EPB * 4 * NP;
  static constexpr int SV = SRES + EPB * 4 * NP;
  static constexpr int SF = SV + ((T == HW_HEX) ? 0 : EPB * 3 * NP);
  static constexpr int SST = SF + EPB * NFP * FLUXW;
  static constexpr int STR = SST + EPB * STG;               // own traces (publishing types)
  static constexpr int SG = STR + ((T == HW_TET) ? 0 : EPB * 4 * NFP);
  static constexpr int SMAT = SG + EPB * X::GEO;
  static constexpr int SOPS = SMAT + EPB * 4;   // hex: D1, x, w, Vend, 1/w
  static constexpr int TOTAL = SOPS + ((T == HW_HEX) ? (N + 1) * (N + 1) + 5 * (N + 1) : 0);
  // ints: element ids, links (x2)
  static constexpr size_t BYTES = sizeof(R) * TOTAL + sizeof(int) * (2 * EPB * NF + EPB);
};

template <int N, int T, typename R>
__device__ __forceinline__ void prologue(const hw_mesh_t& M, const hw_fields_t& Q, const Epi& E,
                                         const int32_t* list, int64_t w0, int ne, R* sm, int* sk,
                                         int* snc, int* sne) {
  using L = Smem<N, T, R>;
  using X = TT<N, T>;
  const hw_type_t& TY = M.t[T];
  const int tid = threadIdx.x;
  if (tid < ne) sk[tid] = list ? list[w0 + tid] : (int)(w0 + tid);
  __syncthreads();
  const R* q = (const R*)Q.p[T];
  for (int i = tid; i < ne * 4 * L::NP; i += NT) {
    const int e = i / (4 * L::NP), r = i - e * 4 * L::NP;
    sm[L::SQ + i] = ldg(q + (size_t)sk[e] * 4 * L::NP + r);
  }
  for (int i = tid; i < ne * X::GEO; i += NT) {
    const int e = i / X::GEO, r = i - e * X::GEO;
    sm[L::SG + i] = ldg((const R*)TY.geo + (size_t)sk[e] * X::GEO + r);
  }
  for (int i = tid; i < ne * 4; i += NT)
    sm[L::SMAT + i] = ldg((const R*)TY.mat + (size_t)sk[i >> 2] * 4 + (i & 3));
  for (int i = tid; i < ne * X::NF; i += NT) {
    const int e = i / X::NF, f = i - e * X::NF;
    const int code = __ldg(TY.nbr_code + (size_t)sk[e] * X::NF + f);
    const int k2 = __ldg(TY.nbr_elem + (size_t)sk[e] * X::NF + f);
    snc[i] = code;
    sne[i] = k2;
  }
  __syncthreads();
  // P1: asynchronous staging (neighbour face values, own traces, LSRK residual)
  const bool sem = M.formulation == HW_SEM;
  stage_neighbours<N, T, R>(M, Q, snc, sne, ne, sm + L::SST, sem);
  if (T != HW_TET && publishes(T, sem)) {
    const R* tr = (const R*)M.tr_in[T];
    for (int i = tid; i < ne * 4 * L::NFP; i += NT) {
      const int e = i / (4 * L::NFP), r = i - e * 4 * L::NFP;
      cp_async(sm + L::STR + i, tr + (size_t)sk[e] * 4 * L::NFP + r);
    }
  }
  if (E.mode == MODE_LSRK) {
    const R* res = (const R*)E.res[T];
    for (int i = tid; i < ne * 4 * L::NP; i += NT) {
      const int e = i / (4 * L::NP), r = i - e * 4 * L::NP;
      cp_async(sm + L::SRES + i, res + (size_t)sk[e] * 4 * L::NP + r);
    }
  }
  cp_async_commit();
}

// epilogue returning the new state value (LSRK / AB; RHS mode returns qv)
template <typename R>
__device__ __forceinline__ R epilogue_q(const Epi& E, int t, size_t idx, R v, R qv, R resv) {
  if (E.mode == MODE_LSRK) {
    const R r = R(E.a) * resv + R(E.dt) * v;
    ((R*)E.res[t])[idx] = r;
    const R qn = qv + R(E.b) * r;
    ((R*)E.qout[t])[idx] = qn;
    return qn;
  }
  if (E.mode == MODE_RHS) {
    ((R*)E.out[t])[idx] = v;
    return qv;
  }
  ((R*)E.out[t])[idx] = v;
  R acc = R(E.c0) * v;
  if (E.nhist > 1) acc += R(E.c1) * ((const R*)E.h1[t])[idx];
  if (E.nhist > 2) acc += R(E.c2) * ((const R*)E.h2[t])[idx];
  const R qn = qv + R(E.dt) * acc;
  ((R*)E.qout[t])[idx] = qn;
  return qn;
}

// epilogue for one value with the LSRK residual prefetched in smem
template <typename R>
__device__ __forceinline__ void epilogue_s(const Epi& E, int t, size_t idx, R v, R qv, R resv) {
  if (E.mode == MODE_LSRK) {
    const R r = R(E.a) * resv + R(E.dt) * v;
    ((R*)E.res[t])[idx] = r;
    ((R*)E.qout[t])[idx] = qv + R(E.b) * r;
  } else {
    epilogue<R>(E, t, idx, v, qv);
  }
}

// ------------------------------------------------------------------ dense types
// tet (nodal, strong), pyramid (semi-nodal quadrature-free, strong GL / skew
// SEM) and affine wedge (LSC-DG, skew).  With constant geometric factors
//   rhs_u_x = -sum_c G[c][x] (A_c p),
//   rhs_p   = -sum_c A_c v_c (strong)  or  +sum_c A_c^T v_c (skew),
//   v_c = sum_x G[c][x] u_x,
// with A_c = D_c (tet, pyramid; hybridwave/dg.py:401-421, 446-463) or
// S_c = V^T W D3_c (wedge: the reference's two cubature passes,
// hybridwave/dg.py:423-444, collapse to it when G and J are constant).
// op[0][c][m][n] = A_c[n][m], op[1][c][m][n] = A_c[m][n].

template <int N, int T, typename R>
__global__ void __launch_bounds__(NT) dense_kernel(hw_mesh_t M, hw_fields_t Q, Epi E,
                                                   const int32_t* __restrict__ list,
                                                   int64_t nwork) {
  using L = Smem<N, T, R>;
  using X = TT<N, T>;
  constexpr int NP = L::NP, NF = L::NF, NFP = L::NFP, EPB = L::EPB, S = L::S;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sm = reinterpret_cast<R*>(smem_raw);
  int* sk = reinterpret_cast<int*>(sm + L::TOTAL);
  int* snc = sk + EPB;
  int* sne = snc + EPB * NF;
  R* sq = sm + L::SQ;
  R* sv = sm + L::SV;
  R* sf = sm + L::SF;
  R* sg = sm + L::SG;
  R* smat = sm + L::SMAT;

  const hw_type_t& TY = M.t[T];
  const int tid = threadIdx.x;
  const int64_t w0 = (int64_t)blockIdx.x * EPB;
  const int ne = (int)((nwork - w0) < EPB ? (nwork - w0) : EPB);
  prologue<N, T, R>(M, Q, E, list, w0, ne, sm, sk, snc, sne);

  const bool skew = TY.form == HW_FORM_SKEW;             // flux form
  const bool vskew = skew || T == HW_WEDGE;              // volume (wedge: always skew)
  // non-affine pyramids (record flag): G and J at every level node from
  // op[8] (K, Np, 10), base-face normals and Js at its points from op[9]
  // (hybridwave/dg.py:446-463, 479-490: J stays inside the skew volume sum
  // and the mass inverse divides by J per node)
  const R* ngeo = (T == HW_PYRAMID) ? (const R*)TY.op[8] : nullptr;
  auto naff = [&](int e) { return T == HW_PYRAMID && sg[e * X::GEO + PY_NAFF] != R(0); };
  // non-affine wedges (Naw): cubature scratch behind the int arrays
  using W8 = Naw<N>;
  const bool naw = T == HW_WEDGE && TY.op[8] != nullptr;
  const R* wgeo = (const R*)TY.op[8];
  const R* wcst = (const R*)TY.op[9];
  // (offset arithmetic on smem_raw itself keeps the pointer in the shared
  // window: LDS / STS instead of generic loads and stores)
  const unsigned cs_off = (unsigned)(((reinterpret_cast<const unsigned char*>(sne + EPB * NF) -
                                       smem_raw) + 15) & ~15);
  R* cs = reinterpret_cast<R*>(smem_raw + cs_off);
  if (T == HW_WEDGE && naw) {
    // trial pass at the volume cubature points: w grad p (incl. the
    // -p grad J / 2J term), w G u, w gJfac . u (hybridwave/dg.py:430-443)
    for (int i = tid; i < ne * W8::NQ; i += NT) {
      const int e = i / W8::NQ, qp = i - e * W8::NQ;
      const R* qe = sq + e * 4 * NP;
      R U[4] = {R(0), R(0), R(0), R(0)}, dc[3] = {R(0), R(0), R(0)};
#pragma unroll 2
      for (int m = 0; m < NP; ++m) {
        const R v = ldg(wcst + m * W8::NQ + qp), pm = qe[m];
        U[0] += v * pm;
        U[1] += v * qe[NP + m];
        U[2] += v * qe[2 * NP + m];
        U[3] += v * qe[3 * NP + m];
        dc[0] += ldg(wcst + (NP + m) * W8::NQ + qp) * pm;
        dc[1] += ldg(wcst + (2 * NP + m) * W8::NQ + qp) * pm;
        dc[2] += ldg(wcst + (3 * NP + m) * W8::NQ + qp) * pm;
      }
      const R* gq = wgeo + (size_t)sk[e] * W8::GW + qp * 12;
      R gl[12];
#pragma unroll
      for (int r = 0; r < 12; ++r) gl[r] = ldg(gq + r);
      R* c = cs + e * W8::CS + qp;
#pragma unroll
      for (int x = 0; x < 3; ++x)
        c[x * W8::NQ] = gl[x] * dc[0] + gl[3 + x] * dc[1] + gl[6 + x] * dc[2] + gl[9 + x] * U[0];
#pragma unroll
      for (int cc = 0; cc < 3; ++cc)
        c[(3 + cc) * W8::NQ] = gl[3 * cc] * U[1] + gl[3 * cc + 1] * U[2] + gl[3 * cc + 2] * U[3];
      c[6 * W8::NQ] = gl[9] * U[1] + gl[10] * U[2] + gl[11] * U[3];
    }
  }

  // contravariant velocity components v_c = sum_x G[c][x] u_x (x J for the
  // non-affine skew pyramid)
  for (int i = tid; i < ne * NP; i += NT) {
    const int e = i / NP, n = i - e * NP;
    // metric in registers (a pointer that may be shared or global would
    // turn every access into a generic load)
    R G[9];
    R sc = R(1);
    if (naff(e)) {
      const R* Gg = ngeo + ((size_t)sk[e] * NP + n) * 10;
#pragma unroll
      for (int a = 0; a < 9; ++a) G[a] = ldg(Gg + a);
      if (vskew) sc = ldg(Gg + 9);
    } else {
#pragma unroll
      for (int a = 0; a < 9; ++a) G[a] = sg[e * X::GEO + a];
    }
    const R* u = sq + e * 4 * NP + NP + n;
#pragma unroll
    for (int c = 0; c < 3; ++c)
      sv[(e * 3 + c) * NP + n] =
          sc * (G[c * 3] * u[0] + G[c * 3 + 1] * u[NP] + G[c * 3 + 2] * u[2 * NP]);
  }
  __syncthreads();

  const R* AT = (const R*)TY.op[0];
  const R* AR = (const R*)TY.op[1];
  R acc[S][4];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = tid + s * NT;
    const int e = i / NP, n = i - e * NP;
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[s][c] = R(0);
    if (T == HW_WEDGE && naw && e < ne) {
      // test pass: R_u = -V^T (w grad p), R_p = sum_c D3_c^T (w G u)_c + V^T (w gJ . u)
      const R* vn = wcst + W8::CVN;
      const R* c = cs + e * W8::CS;
      R a0 = R(0), a1 = R(0), a2 = R(0), a3 = R(0);
#pragma unroll 2
      for (int qp = 0; qp < W8::NQ; ++qp) {
        const R v = ldg(vn + qp * NP + n), dr = ldg(vn + (W8::NQ + qp) * NP + n),
                ds = ldg(vn + (2 * W8::NQ + qp) * NP + n), dt = ldg(vn + (3 * W8::NQ + qp) * NP + n);
        a1 -= v * c[qp];
        a2 -= v * c[W8::NQ + qp];
        a3 -= v * c[2 * W8::NQ + qp];
        a0 += dr * c[3 * W8::NQ + qp] + ds * c[4 * W8::NQ + qp] + dt * c[5 * W8::NQ + qp] +
              v * c[6 * W8::NQ + qp];
      }
      acc[s][0] = a0; acc[s][1] = a1; acc[s][2] = a2; acc[s][3] = a3;
    } else if (e < ne) {
      R div = R(0), dp0 = R(0), dp1 = R(0), dp2 = R(0);
      const R* p = sq + e * 4 * NP;
      const R* v = sv + e * 3 * NP;
      if (vskew) {
#pragma unroll 4
        for (int m = 0; m < NP; ++m) {
          const R pm = p[m];
          dp0 += ldg(AT + (0 * NP + m) * NP + n) * pm;
          dp1 += ldg(AT + (1 * NP + m) * NP + n) * pm;
          dp2 += ldg(AT + (2 * NP + m) * NP + n) * pm;
          div += ldg(AR + (0 * NP + m) * NP + n) * v[m] + ldg(AR + (1 * NP + m) * NP + n) * v[NP + m] +
                 ldg(AR + (2 * NP + m) * NP + n) * v[2 * NP + m];
        }
      } else if (naff(e)) {
        // strong non-affine pyramid: div u(n) = sum_{c,x} G(n)[c][x] (D_c u_x)(n)
        const R* Gn = ngeo + ((size_t)sk[e] * NP + n) * 10;
        R du[3][3] = {{R(0), R(0), R(0)}, {R(0), R(0), R(0)}, {R(0), R(0), R(0)}};
#pragma unroll 2
        for (int m = 0; m < NP; ++m) {
          const R pm = p[m];
          const R a[3] = {ldg(AT + (0 * NP + m) * NP + n), ldg(AT + (1 * NP + m) * NP + n),
                          ldg(AT + (2 * NP + m) * NP + n)};
          dp0 += a[0] * pm;
          dp1 += a[1] * pm;
          dp2 += a[2] * pm;
#pragma unroll
          for (int x = 0; x < 3; ++x) {
            const R um = p[(1 + x) * NP + m];
#pragma unroll
            for (int c = 0; c < 3; ++c) du[x][c] += a[c] * um;
          }
        }
#pragma unroll
        for (int x = 0; x < 3; ++x)
#pragma unroll
          for (int c = 0; c < 3; ++c) div += Gn[3 * c + x] * du[x][c];
      } else {
#pragma unroll 4
        for (int m = 0; m < NP; ++m) {
          const R pm = p[m];
          const R a0 = ldg(AT + (0 * NP + m) * NP + n);
          const R a1 = ldg(AT + (1 * NP + m) * NP + n);
          const R a2 = ldg(AT + (2 * NP + m) * NP + n);
          dp0 += a0 * pm;
          dp1 += a1 * pm;
          dp2 += a2 * pm;
          div += a0 * v[m] + a1 * v[NP + m] + a2 * v[2 * NP + m];
        }
      }
      R G[9];
      R iJ = R(1);
      if (naff(e)) {
        const R* Gg = ngeo + ((size_t)sk[e] * NP + n) * 10;
#pragma unroll
        for (int a = 0; a < 9; ++a) G[a] = ldg(Gg + a);
        iJ = R(1) / ldg(Gg + 9);
      } else {
#pragma unroll
        for (int a = 0; a < 9; ++a) G[a] = sg[e * X::GEO + a];
      }
      acc[s][0] = vskew ? div * iJ : -div;   // affine: J folded into the operators
#pragma unroll
      for (int x = 0; x < 3; ++x) acc[s][1 + x] = -(G[x] * dp0 + G[3 + x] * dp1 + G[6 + x] * dp2);
    }
  }

  cp_async_wait_all();
  __syncthreads();

  // flux at the face points
  const R pen = R(M.penalty_scale);
  for (int i = tid; i < ne * NFP; i += NT) {
    const int e = i / NFP, j = i - e * NFP;
    int jj;
    const int f = face_of_point<N, T>(j, jj);
    if (T == HW_WEDGE && naw && f < 2) continue;   // triangle faces: cubature loop below
    const R* qe = sq + e * 4 * NP;
    R own[4];
    if (T == HW_TET) {
      const int node = __ldg(TY.iop[0] + j);
#pragma unroll
      for (int c = 0; c < 4; ++c) own[c] = qe[c * NP + node];
    } else {   // published traces of the input state
      const R* te = sm + L::STR + e * 4 * NFP + j;
#pragma unroll
      for (int c = 0; c < 4; ++c) own[c] = te[c * NFP];
    }
    const R um[3] = {own[1], own[2], own[3]};
    const R* g = sg + e * X::GEO + X::GF + FS * f;
    R nrm[3] = {g[0], g[1], g[2]};
    R fscale = g[3];
    if (T == HW_PYRAMID && f == 0 && naff(e)) {   // bilinear base: per-point n, Js
      const R* bp = (const R*)TY.op[9] + ((size_t)sk[e] * Dims<N>::NFQ + jj) * 4;
      nrm[0] = ldg(bp); nrm[1] = ldg(bp + 1); nrm[2] = ldg(bp + 2);
      fscale = ldg(bp + 3);
    }
    if (T == HW_WEDGE && naw) {   // bilinear quad face: per-point n, Js/sqrt(J)
      const R* fb = wgeo + (size_t)sk[e] * W8::GW + W8::GF + j * 5;
      nrm[0] = ldg(fb); nrm[1] = ldg(fb + 1); nrm[2] = ldg(fb + 2);
      fscale = ldg(fb + 3);
    }
    const int code = snc[e * NF + f];
    R pp, up[3];
    if (code & HW_NBR_BOUNDARY) {
      pp = -own[0]; up[0] = um[0]; up[1] = um[1]; up[2] = um[2];
    } else {
      R tr[4];
      staged_trace<N, T, R>(M, code, f, jj, sm + L::SST + e * L::STG, tr);
      pp = tr[0]; up[0] = tr[1]; up[1] = tr[2]; up[2] = tr[3];
    }
    R tp, tu, fp, fu;
    penalties(g[4], g[5], pen, tp, tu);
    upwind_flux(own[0], um, pp, up, nrm, tp, tu, skew, fp, fu);
    sf[(e * NFP + j) * 2 + 0] = fp * fscale;
    sf[(e * NFP + j) * 2 + 1] = fu * fscale;
  }
  if (T == HW_WEDGE && naw) {
    // triangle faces at the reference's face cubature points
    const R* LQ = wcst + W8::CLQ;
    R* sfc = cs;   // trial-pass values are dead after the test pass
    for (int i = tid; i < ne * 2 * W8::NQT; i += NT) {
      const int e = i / (2 * W8::NQT), r = i - e * 2 * W8::NQT;
      const int f = r / W8::NQT, qt = r - f * W8::NQT;
      const R* lq = LQ + (f * W8::NQT + qt) * W8::NFN;
      const R* te = sm + L::STR + e * 4 * NFP + f * W8::NFN;   // own polynomial traces
      const int code = snc[e * NF + f];
      const bool bnd = code & HW_NBR_BOUNDARY;
      R own[4] = {R(0), R(0), R(0), R(0)}, nb[4] = {R(0), R(0), R(0), R(0)};
      for (int jj = 0; jj < W8::NFN; ++jj) {
        const R l = ldg(lq + jj);
#pragma unroll
        for (int c = 0; c < 4; ++c) own[c] += l * te[c * NFP + jj];
        if (!bnd) {
          R tr[4];
          staged_trace<N, T, R>(M, code, f, jj, sm + L::SST + e * L::STG, tr);
#pragma unroll
          for (int c = 0; c < 4; ++c) nb[c] += l * tr[c];
        }
      }
      const R* tb = wgeo + (size_t)sk[e] * W8::GW + W8::GT + (f * W8::NQT + qt) * 3;
      const R io = ldg(tb), inb = ldg(tb + 1), sc = ldg(tb + 2);
#pragma unroll
      for (int c = 0; c < 4; ++c) own[c] *= io;
      const R um[3] = {own[1], own[2], own[3]};
      R pp, up[3];
      if (bnd) {
        pp = -own[0]; up[0] = um[0]; up[1] = um[1]; up[2] = um[2];
      } else {
        pp = nb[0] * inb; up[0] = nb[1] * inb; up[1] = nb[2] * inb; up[2] = nb[3] * inb;
      }
      const R* g = sg + e * X::GEO + X::GF + FS * f;
      const R nrm[3] = {g[0], g[1], g[2]};   // planar triangle
      R tp, tu, fp, fu;
      penalties(g[4], g[5], pen, tp, tu);
      upwind_flux(own[0], um, pp, up, nrm, tp, tu, skew, fp, fu);
      sfc[(e * W8::CS) + (f * W8::NQT + qt) * 2 + 0] = fp * sc;
      sfc[(e * W8::CS) + (f * W8::NQT + qt) * 2 + 1] = fu * sc;
    }
  }
  __syncthreads();

  const R* LT = (const R*)TY.op[T == HW_TET ? 1 : 6];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = tid + s * NT;
    const int e = i / NP, n = i - e * NP;
    if (e >= ne) continue;
    const R* fl = sf + e * NFP * 2;
    const R* g = sg + e * X::GEO + X::GF;
    const bool na = naff(e);
    R lift[4] = {R(0), R(0), R(0), R(0)};
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      R tp = R(0), tu = R(0), tux[3] = {R(0), R(0), R(0)};
      const int j0 = X::off(f);
      if (T == HW_WEDGE && naw && f < 2) {   // triangle: Vf^T at the cubature points
        const R* vf = wcst + W8::CVF + f * W8::NQT * NP + n;
        const R* fc = cs + e * W8::CS + f * W8::NQT * 2;
        for (int qt = 0; qt < W8::NQT; ++qt) {
          const R l = ldg(vf + qt * NP);
          tp += l * fc[2 * qt];
          tu += l * fc[2 * qt + 1];
        }
        lift[0] += tp;
        lift[1] += g[FS * f + 0] * tu;
        lift[2] += g[FS * f + 1] * tu;
        lift[3] += g[FS * f + 2] * tu;
        continue;
      }
      // per-point normals: bilinear pyramid base, non-affine wedge quads
      const bool pnrm = (T == HW_PYRAMID && f == 0 && na) || (T == HW_WEDGE && naw);
#pragma unroll 4
      for (int jj = 0; jj < X::cnt(f); ++jj) {
        const int j = j0 + jj;
        const R l = ldg(LT + j * NP + n);
        tp += l * fl[2 * j];
        if (pnrm) {
          const R* bp = T == HW_WEDGE
                            ? wgeo + (size_t)sk[e] * W8::GW + W8::GF + j * 5
                            : (const R*)TY.op[9] + ((size_t)sk[e] * Dims<N>::NFQ + jj) * 4;
          const R lu = l * fl[2 * j + 1];
          tux[0] += lu * ldg(bp); tux[1] += lu * ldg(bp + 1); tux[2] += lu * ldg(bp + 2);
        } else {
          tu += l * fl[2 * j + 1];
        }
      }
      lift[0] += tp;
      if (pnrm) {
        lift[1] += tux[0]; lift[2] += tux[1]; lift[3] += tux[2];
      } else {
        lift[1] += g[FS * f + 0] * tu;
        lift[2] += g[FS * f + 1] * tu;
        lift[3] += g[FS * f + 2] * tu;
      }
    }
    // mass inverse: affine J is folded into the face scale; non-affine
    // pyramids divide by J at the node
    const R liJ = na ? R(1) / ldg(ngeo + ((size_t)sk[e] * NP + n) * 10 + 9) : R(1);
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[s][c] += lift[c] * liJ;
    const R kap = smat[e * 4 + 0], irho = smat[e * 4 + 1];
    const size_t base = (size_t)sk[e] * 4 * NP + n;
    R* qe = sq + e * 4 * NP + n;
    const R* re = sm + L::SRES + e * 4 * NP + n;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const R v = acc[s][c] * (c == 0 ? kap : irho) + frc_at<R>(E, T, base + c * NP);
      const R qn = epilogue_q<R>(E, T, base + c * NP, v, qe[c * NP], re[c * NP]);
      if (T != HW_TET) qe[c * NP] = qn;    // new state, for the published traces
    }
  }
  if (T != HW_TET && E.mode != MODE_RHS && M.tr_out[T] != nullptr) {
    __syncthreads();
    publish_traces<N, T, R>(M, sq, sg, sk, ne, (R*)M.tr_out[T]);
  }
}

// ------------------------------------------------------------------ hex
// Vertex-mapped (trilinear) hex, strong form, GL or GLL(SEM) nodes
// (hybridwave/dg.py:371-399).  Geometry (dx/dr, J, G) is recomputed from
// the 8 vertices at every node and face point instead of being streamed
// from HBM (the reference stores 10 doubles per node).
__constant__ int c_hex_face_verts[6][4] = {
    {0, 4, 7, 3}, {1, 2, 6, 5}, {0, 1, 5, 4}, {2, 3, 7, 6}, {0, 3, 2, 1}, {4, 5, 6, 7}};
__constant__ float c_hex_signs[8][3] = {{-1, -1, -1}, {1, -1, -1}, {1, 1, -1}, {-1, 1, -1},
                                        {-1, -1, 1},  {1, -1, 1},  {1, 1, 1},  {-1, 1, 1}};

template <typename R>
__device__ __forceinline__ R hex_metric(const R* X, R r, R s, R t, R G[9]) {
  R F[9];
#pragma unroll
  for (int a = 0; a < 9; ++a) F[a] = R(0);
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const R sr = R(c_hex_signs[v][0]), ss = R(c_hex_signs[v][1]), st = R(c_hex_signs[v][2]);
    const R fr = R(0.5) * (R(1) + sr * r), fs = R(0.5) * (R(1) + ss * s),
            ft = R(0.5) * (R(1) + st * t);
    const R g0 = R(0.5) * sr * fs * ft, g1 = R(0.5) * ss * fr * ft, g2 = R(0.5) * st * fr * fs;
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      const R xv = X[v * 3 + x];
      F[x * 3 + 0] += xv * g0;   // F[x][c] = dx_x / dr_c
      F[x * 3 + 1] += xv * g1;
      F[x * 3 + 2] += xv * g2;
    }
  }
  const R J = F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) +
              F[2] * (F[3] * F[7] - F[4] * F[6]);
  const R iJ = R(1) / J;
  G[0] = (F[4] * F[8] - F[5] * F[7]) * iJ;
  G[1] = (F[2] * F[7] - F[1] * F[8]) * iJ;
  G[2] = (F[1] * F[5] - F[2] * F[4]) * iJ;
  G[3] = (F[5] * F[6] - F[3] * F[8]) * iJ;
  G[4] = (F[0] * F[8] - F[2] * F[6]) * iJ;
  G[5] = (F[2] * F[3] - F[0] * F[5]) * iJ;
  G[6] = (F[3] * F[7] - F[4] * F[6]) * iJ;
  G[7] = (F[1] * F[6] - F[0] * F[7]) * iJ;
  G[8] = (F[0] * F[4] - F[1] * F[3]) * iJ;
  return J;
}

// node (i, j, k) -> face point c . (i, j, k, 1) of each hex face, per
// formulation and order, in constant memory (hw_prepare uploads the mesh's
// iop[3]): the face index is a compile-time constant of the unrolled lift
// and publish loops, so the coefficients are uniform constant-bank reads
// instead of shared-memory loads (24 per node).
__constant__ int c_hex_spc[2][8][6][4];

#ifndef HW_HEX_NT
#define HW_HEX_NT 128
#endif
// blocks per SM the register allocation must allow (fp64): 7 resident
// blocks (72 registers) for N <= 3; N = 4 (one element per block) runs
// best at 8 (64 registers, 60 B of spills: C4 hex 11.3 -> 11.0 ms; the
// compiler's own choice is 76 registers, 6 blocks, 11.9 ms)
#ifndef HW_HEX_MINB
#define HW_HEX_MINB 0
#endif
template <int N, typename R>
constexpr int hex_minb() {
  return HW_HEX_MINB > 0 ? HW_HEX_MINB : ((sizeof(R) == 8 && N <= 4) ? (N == 4 ? 8 : 7) : 0);
}
#define HW_HEX_BOUNDS __launch_bounds__(HW_HEX_NT, (hex_minb<N, R>()))
// SK: skew form (testing hook); SEM: GLL (spectral-element) nodes, a
// template parameter so the face-point map is compile-time constant-bank
// operands and the formulation branches fold away
// LS: the LSRK stage epilogue (E.mode == MODE_LSRK) compiled in alone
template <int N, typename R, bool SK = false, bool SEM = false, bool LS = false>
__global__ void HW_HEX_BOUNDS hex_kernel(hw_mesh_t M, hw_fields_t Q, Epi E,
                                                 const int32_t* __restrict__ list,
                                                 int64_t nwork) {
  using L = Smem<N, HW_HEX, R, HW_HEX_NT>;
  constexpr int NT = HW_HEX_NT;   // threads per block of this kernel
  using D = Dims<N>;
  constexpr int N1 = D::N1, NP = L::NP, NFQ = D::NFQ, NFP = L::NFP, EPB = L::EPB, S = L::S;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sm = reinterpret_cast<R*>(smem_raw);
  int* sk = reinterpret_cast<int*>(sm + L::TOTAL);
  int* snc = sk + EPB;
  R* sq = sm + L::SQ;
  R* sf = sm + L::SF;
  R* sg = sm + L::SG;
  R* smat = sm + L::SMAT;
  R* sD = sm + L::SOPS;          // D1 (N1 x N1)
  R* sx = sD + N1 * N1;          // 1-D nodes
  R* sw1 = sx + N1;              // 1-D weights
  R* sve = sw1 + N1;             // endpoint rows (2 x N1)
  R* siw1 = sve + 2 * N1;        // 1 / w (1-D)

  const hw_type_t& TY = M.t[HW_HEX];
  constexpr bool sem = SEM;
  const int tid = threadIdx.x;
  const int64_t w0 = (int64_t)blockIdx.x * EPB;
  const int ne = (int)((nwork - w0) < EPB ? (nwork - w0) : EPB);
  if (tid < N1 * N1) sD[tid] = ldg((const R*)TY.op[0] + tid);
  if (tid < 2 * N1) sve[tid] = ldg((const R*)TY.op[1] + tid);
  if (tid < N1) {
    sw1[tid] = ldg((const R*)TY.op[2] + tid);
    siw1[tid] = R(1) / sw1[tid];
    sx[tid] = ldg((const R*)TY.op[4] + tid);
  }
  if (tid < ne) sk[tid] = list ? list[w0 + tid] : (int)(w0 + tid);
  // TMA bulk copies of the element rows: every hex row (state, residual,
  // traces, record, material) is a multiple of 16 bytes, so each element
  // (of a subset list too) is one copy per array.  Group 0: volume inputs;
  // group 1: own traces (GL) and the LSRK residual, waited for by the flux.
  __shared__ __align__(8) uint64_t tbar[2];
  constexpr bool lsrk = LS;
  if (tid == 0) {
    mbar_init(&tbar[0], 1);
    mbar_init(&tbar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  constexpr unsigned ROWB = 4 * NP * sizeof(R), TRB = 4 * NFP * sizeof(R);
  static_assert(ROWB % 16 == 0 && TRB % 16 == 0 && (GEO_HEX * sizeof(R)) % 16 == 0 &&
                    (L::SRES * sizeof(R)) % 16 == 0 && (L::STR * sizeof(R)) % 16 == 0 &&
                    (L::SG * sizeof(R)) % 16 == 0 && (L::SMAT * sizeof(R)) % 16 == 0,
                "hex rows / smem offsets must be 16-byte multiples for the bulk copies");
  if (tid < 32) {
    if (tid == 0) {
      mbar_expect_tx(&tbar[0], ne * (ROWB + (GEO_HEX + 4) * sizeof(R)));
      mbar_expect_tx(&tbar[1], ne * ((sem ? 0u : TRB) + (lsrk ? ROWB : 0u)));
    }
    __syncwarp();
    for (int e = tid; e < ne; e += 32) {
      const size_t k = (size_t)sk[e];
      bulk_load(sq + e * 4 * NP, (const R*)Q.p[HW_HEX] + k * 4 * NP, ROWB, &tbar[0]);
      bulk_load(sg + e * GEO_HEX, (const R*)TY.geo + k * GEO_HEX, GEO_HEX * sizeof(R),
                &tbar[0]);
      bulk_load(smat + e * 4, (const R*)TY.mat + k * 4, 4 * sizeof(R), &tbar[0]);
      if (!sem)
        bulk_load(sm + L::STR + e * 4 * NFP, (const R*)M.tr_in[HW_HEX] + k * 4 * NFP, TRB,
                  &tbar[1]);
      if (lsrk)
        bulk_load(sm + L::SRES + e * 4 * NP, (const R*)E.res[HW_HEX] + k * 4 * NP, ROWB,
                  &tbar[1]);
    }
  }
  for (int i = tid; i < ne * 6; i += NT)
    snc[i] = __ldg(TY.nbr_code + (size_t)sk[i / 6] * 6 + i % 6);
  // the neighbour values at my face points through the host gather index
  {
    constexpr int IT = (EPB * NFP + NT - 1) / NT;
    int gv[IT];
#pragma unroll
    for (int u = 0; u < IT; ++u) {
      const int i = tid + u * NT;
      gv[u] = -1;
      if (i < ne * NFP) gv[u] = __ldg(TY.iop[2] + (size_t)sk[i / NFP] * NFP + i % NFP);
    }
#pragma unroll
    for (int u = 0; u < IT; ++u) {
      const int i = tid + u * NT;
      if (i >= ne * NFP || gv[u] < 0) continue;
      const int e = i / NFP, j = i - e * NFP;
      const int t2 = HW_NBR_TYPE(__ldg(TY.nbr_code + (size_t)sk[e] * 6 + j / NFQ));
      const R* src;
      int stride;
      if (publishes(t2, sem)) {
        src = (const R*)M.tr_in[t2];
        stride = nfp_of<N>(t2);
      } else {
        src = (const R*)Q.p[HW_HEX];
        stride = NP;
      }
      src += gv[u];
      R* dst = sm + L::SST + e * 4 * NFP + j;
#pragma unroll
      for (int c = 0; c < 4; ++c) cp_async(dst + c * NFP, src + c * stride);
    }
  }
  cp_async_commit();
  mbar_wait(&tbar[0], 0);
  __syncthreads();     // snc

  // skew form (forms_override testing hook, hybridwave/dg.py:392-398): the
  // pressure term is sum_c D^T (w3 J v_c), v_c = sum_x G[c][x] u_x, formed
  // here in the flux storage (written only after the volume pass)
  constexpr bool skew = SK;
  R* spre = sf;   // [e][c][node]
  static_assert(3 * NP <= 4 * NFP, "the volume scratch lives in the flux storage");
  if (!skew) {
    // affine elements: div u = sum_c d_c V_c with the contravariant velocity
    // V_c = sum_x G[c][x] u_x (G constant), so the volume pass differentiates
    // two quantities per direction (p, V_c) instead of four
    for (int i = tid; i < ne * NP; i += NT) {
      const int e = i / NP, n = i - e * NP;
      const R* Xe = sg + e * GEO_HEX;
      if (Xe[HX_AFF] == R(0)) continue;
      const R* u = sq + e * 4 * NP + n;
      const R u0 = u[NP], u1 = u[2 * NP], u2 = u[3 * NP];
#pragma unroll
      for (int c = 0; c < 3; ++c)
        spre[(e * 3 + c) * NP + n] =
            Xe[HX_G + 3 * c] * u0 + Xe[HX_G + 3 * c + 1] * u1 + Xe[HX_G + 3 * c + 2] * u2;
    }
    __syncthreads();
  } else {
    for (int i = tid; i < ne * NP; i += NT) {
      const int e = i / NP, n = i - e * NP;
      const int ii = n / (N1 * N1), jj = (n / N1) % N1, kk = n % N1;
      const R* Xe = sg + e * GEO_HEX;
      R G[9], J;
      if (Xe[HX_AFF] != R(0)) {
#pragma unroll
        for (int a = 0; a < 9; ++a) G[a] = Xe[HX_G + a];
        J = Xe[HX_J];
      } else {
        J = hex_metric<R>(Xe, sx[ii], sx[jj], sx[kk], G);
      }
      const R wJ = sw1[ii] * sw1[jj] * sw1[kk] * J;
      const R* u = sq + e * 4 * NP + n;
#pragma unroll
      for (int c = 0; c < 3; ++c)
        spre[(e * 3 + c) * NP + n] =
            wJ * (G[3 * c] * u[NP] + G[3 * c + 1] * u[2 * NP] + G[3 * c + 2] * u[3 * NP]);
    }
    __syncthreads();
  }

  R acc[S][4], minv[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = tid + s * NT;
    const int e = i / NP, n = i - e * NP;
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[s][c] = R(0);
    minv[s] = R(0);
    if (e < ne) {
      const int ii = n / (N1 * N1), jj = (n / N1) % N1, kk = n % N1;
      const R* Xe = sg + e * GEO_HEX;
      if (!skew && Xe[HX_AFF] != R(0)) {
        const R* u = sq + e * 4 * NP;
        const R* V = spre + e * 3 * NP;
        R a0 = R(0), a1 = R(0), a2 = R(0), div = R(0);
#pragma unroll
        for (int l = 0; l < N1; ++l) {
          const R dr = sD[ii * N1 + l], ds = sD[jj * N1 + l], dt = sD[kk * N1 + l];
          const int nr = (l * N1 + jj) * N1 + kk, ns = (ii * N1 + l) * N1 + kk,
                    nt = (ii * N1 + jj) * N1 + l;
          a0 += dr * u[nr];
          a1 += ds * u[ns];
          a2 += dt * u[nt];
          div += dr * V[nr] + ds * V[NP + ns] + dt * V[2 * NP + nt];
        }
#pragma unroll
        for (int x = 0; x < 3; ++x)
          acc[s][1 + x] = -(Xe[HX_G + x] * a0 + Xe[HX_G + 3 + x] * a1 + Xe[HX_G + 6 + x] * a2);
        acc[s][0] = -div;
        minv[s] = siw1[ii] * siw1[jj] * siw1[kk] * Xe[HX_IJ];
        continue;
      }
      R d[4][3];
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        const R* u = sq + (e * 4 + f) * NP;
        R a0 = R(0), a1 = R(0), a2 = R(0);
#pragma unroll
        for (int l = 0; l < N1; ++l) {
          a0 += sD[ii * N1 + l] * u[(l * N1 + jj) * N1 + kk];
          a1 += sD[jj * N1 + l] * u[(ii * N1 + l) * N1 + kk];
          a2 += sD[kk * N1 + l] * u[(ii * N1 + jj) * N1 + l];
        }
        d[f][0] = a0; d[f][1] = a1; d[f][2] = a2;
      }
      R G[9];
      R iJ;
      if (Xe[HX_AFF] != R(0)) {       // affine: constant metric from the record
#pragma unroll
        for (int a = 0; a < 9; ++a) G[a] = Xe[HX_G + a];
        iJ = Xe[HX_IJ];
      } else {
        iJ = R(1) / hex_metric<R>(Xe, sx[ii], sx[jj], sx[kk], G);
      }
      R div = R(0);
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        acc[s][1 + x] = -(G[x] * d[0][0] + G[3 + x] * d[0][1] + G[6 + x] * d[0][2]);
        div += G[x] * d[1 + x][0] + G[3 + x] * d[1 + x][1] + G[6 + x] * d[1 + x][2];
      }
      acc[s][0] = -div;
      minv[s] = siw1[ii] * siw1[jj] * siw1[kk] * iJ;
      if (skew) {
        const R* pr = spre + e * 3 * NP;
        R a = R(0);
#pragma unroll
        for (int l = 0; l < N1; ++l)
          a += sD[l * N1 + ii] * pr[(l * N1 + jj) * N1 + kk] +
               sD[l * N1 + jj] * pr[NP + (ii * N1 + l) * N1 + kk] +
               sD[l * N1 + kk] * pr[2 * NP + (ii * N1 + jj) * N1 + l];
        acc[s][0] = a * minv[s];
      }
    }
  }

  cp_async_wait_all();
  mbar_wait(&tbar[1], 0);
  __syncthreads();

  const R pen = R(M.penalty_scale);
  for (int i = tid; i < ne * NFP; i += NT) {
    const int e = i / NFP, j = i - e * NFP;
    const int f = j / NFQ, jj = j - f * NFQ;
    const R* qe = sq + e * 4 * NP;
    R own[4];
    if (sem) {
      const int* tab = TY.iop[0] + 3 * j;
      const int base = __ldg(tab), stride = __ldg(tab + 1), end = __ldg(tab + 2);
      const int node = base + (end ? N : 0) * stride;
#pragma unroll
      for (int c = 0; c < 4; ++c) own[c] = qe[c * NP + node];
    } else {   // GL: published traces of the input state
      const R* te = sm + L::STR + e * 4 * NFP + j;
#pragma unroll
      for (int c = 0; c < 4; ++c) own[c] = te[c * NFP];
    }
    // face geometry at (xi, eta) = (x[a], x[b]) from the 4 face vertices
    const int a = jj / N1, b = jj - a * N1;
    const R xi = sx[a], eta = sx[b];
    const R* Xv = sg + e * GEO_HEX;
    R nrm[3], Js;
    if (Xv[HX_AFF] != R(0)) {
      const R* fr = Xv + HX_F + 4 * f;
      nrm[0] = fr[0]; nrm[1] = fr[1]; nrm[2] = fr[2];
      Js = fr[3];
    } else {
    R t1[3], t2[3];
    {
      const R g1[4] = {-(R(1) - eta), (R(1) - eta), (R(1) + eta), -(R(1) + eta)};
      const R g2[4] = {-(R(1) - xi), -(R(1) + xi), (R(1) + xi), (R(1) - xi)};
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        R s1 = R(0), s2 = R(0);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const R xv = Xv[c_hex_face_verts[f][v] * 3 + x];
          s1 += g1[v] * xv;
          s2 += g2[v] * xv;
        }
        t1[x] = R(0.25) * s1;
        t2[x] = R(0.25) * s2;
      }
    }
    const R nv[3] = {t1[1] * t2[2] - t1[2] * t2[1], t1[2] * t2[0] - t1[0] * t2[2],
                     t1[0] * t2[1] - t1[1] * t2[0]};
    Js = sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
    nrm[0] = nv[0] / Js; nrm[1] = nv[1] / Js; nrm[2] = nv[2] / Js;
    }
    const R wJs = sw1[a] * sw1[b] * Js;
    const R um[3] = {own[1], own[2], own[3]};
    const int code = snc[e * 6 + f];
    R pp, up[3];
    if (code & HW_NBR_BOUNDARY) {
      pp = -own[0]; up[0] = um[0]; up[1] = um[1]; up[2] = um[2];
    } else {   // neighbour values staged in my point order
      const R* se = sm + L::SST + e * 4 * NFP + j;
      pp = se[0]; up[0] = se[NFP]; up[1] = se[2 * NFP]; up[2] = se[3 * NFP];
    }
    R tp, tu, fp, fu;
    penalties(Xv[HX_Z + 2 * f], Xv[HX_Z + 2 * f + 1], pen, tp, tu);
    upwind_flux(own[0], um, pp, up, nrm, tp, tu, SK, fp, fu);
    R* o = sf + e * 4 * NFP + j;        // [field][face point]: conflict-free
    o[0] = fp * wJs;
    o[NFP] = nrm[0] * fu * wJs;
    o[2 * NFP] = nrm[1] * fu * wJs;
    o[3 * NFP] = nrm[2] * fu * wJs;
  }
  __syncthreads();

#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = tid + s * NT;
    const int e = i / NP, n = i - e * NP;
    if (e >= ne) continue;
    const int idx[3] = {n / (N1 * N1), (n / N1) % N1, n % N1};
    const R* fl = sf + e * NFP * 4;
    R lift[4] = {R(0), R(0), R(0), R(0)};
    // (hex: fl is [field][face point])
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      const int axis = f >> 1, end = f & 1;
      const int l = idx[axis];
      R w;
      if (sem) {
        if (l != (end ? N : 0)) continue;
        w = R(1);
      } else {
        w = sve[end * N1 + l];
      }
      const int* cf = c_hex_spc[SEM ? 1 : 0][N][f];
      const int pt = cf[0] * idx[0] + cf[1] * idx[1] + cf[2] * idx[2] + cf[3];
      const R* o = fl + f * NFQ + pt;
#pragma unroll
      for (int c = 0; c < 4; ++c) lift[c] += w * o[c * NFP];
    }
    // only the surface term carries the mass inverse 1/(w3 J): the volume
    // term above is already the cancelled form -grad p, -div u
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[s][c] += lift[c] * minv[s];
    const R kap = smat[e * 4 + 0], irho = smat[e * 4 + 1];
    const size_t base = (size_t)sk[e] * 4 * NP + n;
    R* qe = sq + e * 4 * NP + n;
    R* re = sm + L::SRES + e * 4 * NP + n;
    // results into the staged rows (q_out over q; the residual / rhs / new
    // slope over the residual row), written back by bulk stores below
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const R v = acc[s][c] * (c == 0 ? kap : irho) + frc_at<R>(E, HW_HEX, base + c * NP);
      const R qv = qe[c * NP];
      if (lsrk) {
        const R r = R(E.a) * re[c * NP] + R(E.dt) * v;
        re[c * NP] = r;
        qe[c * NP] = qv + R(E.b) * r;
      } else if (E.mode == MODE_RHS) {
        re[c * NP] = v;
      } else {
        R a = R(E.c0) * v;
        if (E.nhist > 1) a += R(E.c1) * ((const R*)E.h1[HW_HEX])[base + c * NP];
        if (E.nhist > 2) a += R(E.c2) * ((const R*)E.h2[HW_HEX])[base + c * NP];
        re[c * NP] = v;
        qe[c * NP] = qv + R(E.dt) * a;
      }
    }
  }
  const bool pub = !sem && E.mode != MODE_RHS && M.tr_out[HW_HEX] != nullptr;
  if (pub) {
    __syncthreads();
    // GL hex traces of the new state: one thread per (element, axis, line)
    // reads the line once and interpolates to both end faces of the axis;
    // into the (dead) own-trace rows, bulk-stored with the state rows
    // (when the (element, axis) pairs fit one warp each, every warp takes
    // one axis: its loads and its face-row stores then stay within one
    // contiguous block of words, without the bank conflicts of a warp
    // straddling two axes)
    constexpr int LW = (NFQ > 16 && NFQ <= 32 && EPB * 3 * 32 <= NT) ? 32 : NFQ;
    for (int it = tid; it < ne * 3 * LW; it += NT) {
      const int e = it / (3 * LW), r = it - e * 3 * LW;
      const int a = r / LW, uv = r - a * LW, u = uv / N1, v = uv - u * N1;
      if (uv >= NFQ) continue;
      // base node (axis index 0) and stride along the axis
      const int ii = a == 0 ? 0 : u, jj = a == 0 ? u : (a == 1 ? 0 : v), kk = a == 2 ? 0 : v;
      const int base = (ii * N1 + jj) * N1 + kk;
      const int stride = a == 0 ? N1 * N1 : (a == 1 ? N1 : 1);
      const R* qe = sq + e * 4 * NP + base;
      R t0[4] = {R(0), R(0), R(0), R(0)}, t1[4] = {R(0), R(0), R(0), R(0)};
#pragma unroll
      for (int l = 0; l < N1; ++l) {
        const R w0 = sve[l], w1 = sve[N1 + l];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const R x = qe[c * NP + l * stride];
          t0[c] += w0 * x;
          t1[c] += w1 * x;
        }
      }
      R* o = sm + L::STR + e * 4 * NFP;
#pragma unroll
      for (int end = 0; end < 2; ++end) {
        const int f = 2 * a + end;
        const int* cf = c_hex_spc[SEM ? 1 : 0][N][f];
        const int pt = cf[0] * ii + cf[1] * jj + cf[2] * kk + cf[3];
#pragma unroll
        for (int c = 0; c < 4; ++c) o[c * NFP + f * NFQ + pt] = end ? t1[c] : t0[c];
      }
    }
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (tid < 32) {
    R* dq = E.mode == MODE_RHS ? nullptr : (R*)E.qout[HW_HEX];
    R* dr = (R*)(lsrk ? E.res[HW_HEX] : E.out[HW_HEX]);
    for (int e = tid; e < ne; e += 32) {
      const size_t k = (size_t)sk[e];
      bulk_store(dr + k * 4 * NP, sm + L::SRES + e * 4 * NP, ROWB);
      if (dq) bulk_store(dq + k * 4 * NP, sq + e * 4 * NP, ROWB);
      if (pub) bulk_store((R*)M.tr_out[HW_HEX] + k * 4 * NFP, sm + L::STR + e * 4 * NFP, TRB);
    }
    bulk_commit();
    bulk_wait_read();
  }
}

// Discrete energy U^T M U with material weights (hybridwave/dg.py:655-674):
// p / kappa + rho |u|^2, mass: hex w3 J (per node), tet J M_ref, pyramid J,
// wedge identity (LSC basis).  One thread per (element, node); block sums
// accumulate into out[T] with a double atomicAdd.
// J of a trilinear hex at node (a, b, c) (out of line: the energy kernel's
// unrolled node loop would otherwise inline one metric per node it holds)
template <typename R>
__device__ __noinline__ double hex_J_at(const R* g, const R* x1, int a, int b, int c) {
  R G[9];
  return (double)hex_metric<R>(g, x1[a], x1[b], x1[c], G);
}

template <int N, int T, typename R>
__global__ void __launch_bounds__(256) energy_kernel(hw_mesh_t M, hw_fields_t Q, double* out,
                                                     int64_t K) {
  // one warp per element (lanes over the nodes: coalesced state reads, the
  // element's record and material read once); tets stage the element rows
  // in shared memory for (M_ref u)_n with M_ref resident per block
  using X = TT<N, T>;
  using D = Dims<N>;
  constexpr int NP = X::NP, NW = 8;
  const hw_type_t& TY = M.t[T];
  const R* q = (const R*)Q.p[T];
  const R* geo = (const R*)TY.geo;
  const R* mat = (const R*)TY.mat;
  constexpr bool SMEM_M = T == HW_TET && NP * NP <= 4096;   // N <= 5: M_ref in smem
  __shared__ double sM[SMEM_M ? NP * NP : 1];
  __shared__ double sqe[(T == HW_TET) ? NW * 4 * NP : 1];
  __shared__ double sw1[D::N1];
  if (SMEM_M)
    for (int i = threadIdx.x; i < NP * NP; i += blockDim.x) sM[i] = (double)ldg((const R*)TY.op[4] + i);
  if (T == HW_HEX && threadIdx.x < D::N1) sw1[threadIdx.x] = (double)ldg((const R*)TY.op[2] + threadIdx.x);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * NW + warp; e < K; e += (int64_t)gridDim.x * NW) {
    const R* qe = q + e * 4 * NP;
    const double wp = 1.0 / (double)mat[e * 4 + 0], wu = 1.0 / (double)mat[e * 4 + 1];
    const R* g = geo + e * X::GEO;
    bool aff = true;
    double we = 1.0;   // element-constant mass weight (J; wedge 1)
    if (T == HW_HEX) {
      aff = g[HX_AFF] != R(0);
      if (aff) we = (double)g[HX_J];
    } else if (T == HW_PYRAMID && g[PY_NAFF] != R(0)) {
      aff = false;
    } else if (T != HW_WEDGE) {
      const double det = (double)g[0] * ((double)g[4] * g[8] - (double)g[5] * g[7]) -
                         (double)g[1] * ((double)g[3] * g[8] - (double)g[5] * g[6]) +
                         (double)g[2] * ((double)g[3] * g[7] - (double)g[4] * g[6]);
      we = 1.0 / det;   // G = dr/dx: det G = 1/J
    }
    double* sq = sqe + warp * 4 * NP;
    constexpr int IT = (NP + 31) / 32;
    double qv[IT][4];          // this lane's node values, all loads in flight at once
#pragma unroll
    for (int u = 0; u < IT; ++u) {
      const int n = lane + 32 * u;
#pragma unroll
      for (int c = 0; c < 4; ++c) qv[u][c] = n < NP ? (double)qe[c * NP + n] : 0.0;
    }
    if (T == HW_TET) {
#pragma unroll
      for (int u = 0; u < IT; ++u) {
        const int n = lane + 32 * u;
        if (n < NP)
#pragma unroll
          for (int c = 0; c < 4; ++c) sq[c * NP + n] = qv[u][c];
      }
      __syncwarp();
    }
#pragma unroll
    for (int u = 0; u < IT; ++u) {
      const int n = lane + 32 * u;
      if (n >= NP) break;
      double w = we;
      if (T == HW_HEX) {
        const int a = n / (D::N1 * D::N1), b = (n / D::N1) % D::N1, c = n % D::N1;
        const double J = aff ? we : hex_J_at<R>(g, (const R*)TY.op[4], a, b, c);
        w = sw1[a] * sw1[b] * sw1[c] * J;
      } else if (T == HW_PYRAMID && !aff) {
        w = (double)ldg((const R*)TY.op[8] + ((size_t)e * NP + n) * 10 + 9);   // J at the node
      }
      double s = 0.0;
      if constexpr (T == HW_TET) {   // (M_ref u)_n for the four fields at once
        double mv[4] = {0.0, 0.0, 0.0, 0.0};
        const R* Mr = (const R*)TY.op[4] + n * NP;
#pragma unroll 5
        for (int j = 0; j < NP; ++j) {
          const double m = SMEM_M ? sM[n * NP + j] : (double)ldg(Mr + j);
#pragma unroll
          for (int c = 0; c < 4; ++c) mv[c] += m * sq[c * NP + j];
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) s += (c == 0 ? wp : wu) * qv[u][c] * mv[c];
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) s += (c == 0 ? wp : wu) * qv[u][c] * qv[u][c];
      }
      acc += w * s;
    }
    if (T == HW_TET) __syncwarp();
  }
  // block reduction
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) atomicAdd(out + T, acc);
  }
}

// Face traces of q for a publishing type (hw_traces): EPB elements per block.
template <int N, int T, typename R>
__global__ void __launch_bounds__(NT) trace_kernel(hw_mesh_t M, hw_fields_t Q, hw_fields_t TR,
                                                   const int32_t* __restrict__ list,
                                                   int64_t nwork) {
  using X = TT<N, T>;
  constexpr int NP = X::NP;
  constexpr int EPB = (NT / NP) > 0 ? (NT / NP) : 1;
  __shared__ R sq[EPB * 4 * NP];
  __shared__ R sg[EPB * X::GEO];
  __shared__ int sk[EPB];
  const int tid = threadIdx.x;
  const int64_t w0 = (int64_t)blockIdx.x * EPB;
  const int ne = (int)((nwork - w0) < EPB ? (nwork - w0) : EPB);
  if (tid < ne) sk[tid] = list ? list[w0 + tid] : (int)(w0 + tid);
  __syncthreads();
  const R* q = (const R*)Q.p[T];
  for (int i = tid; i < ne * 4 * NP; i += NT) {
    const int e = i / (4 * NP), r = i - e * 4 * NP;
    sq[i] = ldg(q + (size_t)sk[e] * 4 * NP + r);
  }
  for (int i = tid; i < ne * X::GEO; i += NT) {
    const int e = i / X::GEO, r = i - e * X::GEO;
    sg[i] = ldg((const R*)M.t[T].geo + (size_t)sk[e] * X::GEO + r);
  }
  __syncthreads();
  publish_traces<N, T, R>(M, sq, sg, sk, ne, (R*)TR.p[T]);
}

}  // namespace hw
