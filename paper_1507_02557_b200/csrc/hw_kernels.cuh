// Fused per-element-type RHS + time-update kernels (sm_100a).
//
// One launch per element type per stage.  A block owns EPB elements and
// runs, with a block barrier between phases:
//   load      q (4 x Np per element) and the per-element geometry record
//   volume    strong/skew volume term with the mass inverse folded out
//             (SURVEY.md 8a "algebraic cancellations")
//   flux      own trace, neighbour trace (read from the neighbour's input
//             state), upwind flux, scaled by the face Jacobian
//   lift      face-to-volume lift, mass inverse, material scaling, and the
//             epilogue (RHS / LSRK stage / AB step)
// Reference data flow: hybridwave/dg.py:299-506.
#pragma once
#include "hw_common.cuh"

namespace hw {

// ------------------------------------------------------------------ tet
// Strong form (both formulations, hybridwave/dg.py:34-37, 401-421):
//   rhs_p = -sum_c D_c (sum_x G[c][x] u_x),  rhs_u_x = -sum_c G[c][x] D_c p
// then + (Js_f/J) LIFT_f flux_f, LIFT = invM_ref Vf^T W L (nodal faces).
template <int N, typename R>
struct TetK {
  using D = Dims<N>;
  static constexpr int NP = D::NP_TET, NFN = D::NFN, NFP = D::NFP_TET;
  static constexpr int EPB = (NT / NP) > 0 ? (NT / NP) : 1;
  static constexpr int S = (EPB * NP + NT - 1) / NT;
  static constexpr int SQ = 0, SV = SQ + EPB * 4 * NP, SF = SV + EPB * 3 * NP,
                       SG = SF + EPB * NFP * 2, SM = SG + EPB * GEO_TET,
                       SMEM = SM + EPB * 4;
};

template <int N, typename R>
__global__ void __launch_bounds__(NT) tet_kernel(hw_mesh_t M, hw_fields_t Q, Epi E,
                                                 const int32_t* __restrict__ list,
                                                 int64_t nwork) {
  using K_ = TetK<N, R>;
  constexpr int NP = K_::NP, NFN = K_::NFN, NFP = K_::NFP, EPB = K_::EPB, S = K_::S;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sm = reinterpret_cast<R*>(smem_raw);
  R* sq = sm + K_::SQ;
  R* sv = sm + K_::SV;
  R* sf = sm + K_::SF;
  R* sg = sm + K_::SG;
  R* smat = sm + K_::SM;
  __shared__ int sk[EPB];

  const hw_type_t& T = M.t[HW_TET];
  const int tid = threadIdx.x;
  const int64_t w0 = (int64_t)blockIdx.x * EPB;
  const int ne = (int)((nwork - w0) < EPB ? (nwork - w0) : EPB);
  if (tid < ne) sk[tid] = list ? list[w0 + tid] : (int)(w0 + tid);
  __syncthreads();

  const R* q = (const R*)Q.p[HW_TET];
  for (int i = tid; i < ne * 4 * NP; i += NT) {
    const int e = i / (4 * NP), r = i - e * 4 * NP;
    sq[i] = ldg(q + (size_t)sk[e] * 4 * NP + r);
  }
  for (int i = tid; i < ne * GEO_TET; i += NT) {
    const int e = i / GEO_TET, r = i - e * GEO_TET;
    sg[i] = ldg((const R*)T.geo + (size_t)sk[e] * GEO_TET + r);
  }
  for (int i = tid; i < ne * 4; i += NT) {
    sm[K_::SM + i] = ldg((const R*)T.mat + (size_t)sk[i / 4] * 4 + (i & 3));
  }
  __syncthreads();

  // contravariant velocity components v_c = sum_x G[c][x] u_x
  for (int i = tid; i < ne * NP; i += NT) {
    const int e = i / NP, n = i - e * NP;
    const R* G = sg + e * GEO_TET;
    const R* u = sq + e * 4 * NP + NP + n;
#pragma unroll
    for (int c = 0; c < 3; ++c)
      sv[(e * 3 + c) * NP + n] = G[c * 3 + 0] * u[0] + G[c * 3 + 1] * u[NP] + G[c * 3 + 2] * u[2 * NP];
  }
  __syncthreads();

  R acc[S][4];
  const R* DT = (const R*)T.op[0];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = tid + s * NT;
    const int e = i / NP, n = i - e * NP;
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[s][c] = R(0);
    if (e < ne) {
      R div = R(0), dp[3] = {R(0), R(0), R(0)};
      const R* p = sq + e * 4 * NP;
      const R* v = sv + e * 3 * NP;
#pragma unroll 4
      for (int m = 0; m < NP; ++m) {
        const R pm = p[m];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const R d = ldg(DT + (c * NP + m) * NP + n);
          div += d * v[c * NP + m];
          dp[c] += d * pm;
        }
      }
      const R* G = sg + e * GEO_TET;
      acc[s][0] = -div;
#pragma unroll
      for (int x = 0; x < 3; ++x)
        acc[s][1 + x] = -(G[x] * dp[0] + G[3 + x] * dp[1] + G[6 + x] * dp[2]);
    }
  }

  // face flux at the tet face nodes
  const R pen = R(M.penalty_scale);
  for (int i = tid; i < ne * NFP; i += NT) {
    const int e = i / NFP, j = i - e * NFP;
    const int f = j / NFN, jj = j - f * NFN;
    const int k = sk[e];
    const int node = __ldg(T.iop[0] + j);
    const R* qe = sq + e * 4 * NP;
    const R pm = qe[node];
    const R um[3] = {qe[NP + node], qe[2 * NP + node], qe[3 * NP + node]};
    const R* g = sg + e * GEO_TET + 9 + 4 * f;
    const R nrm[3] = {g[0], g[1], g[2]};
    const int code = __ldg(T.nbr_code + (size_t)k * NF_TET + f);
    const R zm = smat[e * 4 + 2];
    R pp, up[3], zp;
    if (code & HW_NBR_BOUNDARY) {
      pp = -pm; up[0] = um[0]; up[1] = um[1]; up[2] = um[2]; zp = zm;
    } else {
      const int k2 = __ldg(T.nbr_elem + (size_t)k * NF_TET + f);
      R tr[4];
      neighbour_trace<N, R>(M, Q, code, k2, jj, true, tr);
      pp = tr[0]; up[0] = tr[1]; up[1] = tr[2]; up[2] = tr[3];
      zp = neighbour_z<R>(M, code, k2);
    }
    R tp, tu, fp, fu;
    penalties(zm, zp, pen, tp, tu);
    upwind_flux(pm, um, pp, up, nrm, tp, tu, T.form == HW_FORM_SKEW, fp, fu);
    sf[(e * NFP + j) * 2 + 0] = fp * g[3];
    sf[(e * NFP + j) * 2 + 1] = fu * g[3];
  }
  __syncthreads();

  const R* LT = (const R*)T.op[1];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = tid + s * NT;
    const int e = i / NP, n = i - e * NP;
    if (e >= ne) continue;
    const R* fl = sf + e * NFP * 2;
    const R* g = sg + e * GEO_TET + 9;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      R tp = R(0), tu = R(0);
#pragma unroll 4
      for (int jj = 0; jj < NFN; ++jj) {
        const int j = f * NFN + jj;
        const R l = ldg(LT + j * NP + n);
        tp += l * fl[2 * j];
        tu += l * fl[2 * j + 1];
      }
      acc[s][0] += tp;
      acc[s][1] += g[4 * f + 0] * tu;
      acc[s][2] += g[4 * f + 1] * tu;
      acc[s][3] += g[4 * f + 2] * tu;
    }
    const R kap = smat[e * 4 + 0], irho = smat[e * 4 + 1];
    const size_t base = (size_t)sk[e] * 4 * NP + n;
    const R* qe = sq + e * 4 * NP + n;
    epilogue<R>(E, HW_TET, base, acc[s][0] * kap, qe[0]);
#pragma unroll
    for (int c = 1; c < 4; ++c) epilogue<R>(E, HW_TET, base + c * NP, acc[s][c] * irho, qe[c * NP]);
  }
}

// ------------------------------------------------------------------ pyramid
// Quadrature-free semi-nodal pyramid (hybridwave/dg.py:446-463), affine:
//   strong (GL):  rhs_p = -sum_c D_c v_c
//   skew (SEM):   rhs_p = +sum_c D_c^T v_c        (v_c = sum_x G[c][x] u_x)
//   rhs_u_x = -sum_c G[c][x] D_c p
// surface: (Js/J) LIFT flux with LIFT = Vf^T W L.
template <int N, typename R>
struct PyrK {
  using D = Dims<N>;
  static constexpr int NP = D::NP_PYR, NFN = D::NFN, NFQ = D::NFQ, NFP = D::NFP_PYR;
  static constexpr int EPB = (NT / NP) > 0 ? (NT / NP) : 1;
  static constexpr int S = (EPB * NP + NT - 1) / NT;
  static constexpr int SQ = 0, SV = SQ + EPB * 4 * NP, SF = SV + EPB * 3 * NP,
                       SG = SF + EPB * NFP * 2, SM = SG + EPB * GEO_PYR,
                       SMEM = SM + EPB * 4;
};

template <int N, typename R>
__global__ void __launch_bounds__(NT) pyr_kernel(hw_mesh_t M, hw_fields_t Q, Epi E,
                                                 const int32_t* __restrict__ list,
                                                 int64_t nwork) {
  using K_ = PyrK<N, R>;
  constexpr int NP = K_::NP, NFN = K_::NFN, NFQ = K_::NFQ, NFP = K_::NFP, EPB = K_::EPB,
                S = K_::S;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sm = reinterpret_cast<R*>(smem_raw);
  R* sq = sm + K_::SQ;
  R* sv = sm + K_::SV;
  R* sf = sm + K_::SF;
  R* sg = sm + K_::SG;
  R* smat = sm + K_::SM;
  __shared__ int sk[EPB];

  const hw_type_t& T = M.t[HW_PYRAMID];
  const int tid = threadIdx.x;
  const int64_t w0 = (int64_t)blockIdx.x * EPB;
  const int ne = (int)((nwork - w0) < EPB ? (nwork - w0) : EPB);
  if (tid < ne) sk[tid] = list ? list[w0 + tid] : (int)(w0 + tid);
  __syncthreads();

  const R* q = (const R*)Q.p[HW_PYRAMID];
  for (int i = tid; i < ne * 4 * NP; i += NT) {
    const int e = i / (4 * NP), r = i - e * 4 * NP;
    sq[i] = ldg(q + (size_t)sk[e] * 4 * NP + r);
  }
  for (int i = tid; i < ne * GEO_PYR; i += NT) {
    const int e = i / GEO_PYR, r = i - e * GEO_PYR;
    sg[i] = ldg((const R*)T.geo + (size_t)sk[e] * GEO_PYR + r);
  }
  for (int i = tid; i < ne * 4; i += NT)
    smat[i] = ldg((const R*)T.mat + (size_t)sk[i / 4] * 4 + (i & 3));
  __syncthreads();

  for (int i = tid; i < ne * NP; i += NT) {
    const int e = i / NP, n = i - e * NP;
    const R* G = sg + e * GEO_PYR;
    const R* u = sq + e * 4 * NP + NP + n;
#pragma unroll
    for (int c = 0; c < 3; ++c)
      sv[(e * 3 + c) * NP + n] = G[c * 3 + 0] * u[0] + G[c * 3 + 1] * u[NP] + G[c * 3 + 2] * u[2 * NP];
  }
  __syncthreads();

  const bool skew = T.form == HW_FORM_SKEW;
  R acc[S][4];
  const R* DT = (const R*)T.op[0];   // DT[c][m][n] = D_c[n][m]
  const R* DR = (const R*)T.op[1];   // DR[c][m][n] = D_c[m][n]
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = tid + s * NT;
    const int e = i / NP, n = i - e * NP;
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[s][c] = R(0);
    if (e < ne) {
      R div = R(0), dp[3] = {R(0), R(0), R(0)};
      const R* p = sq + e * 4 * NP;
      const R* v = sv + e * 3 * NP;
      const R* DV = skew ? DR : DT;
#pragma unroll 2
      for (int m = 0; m < NP; ++m) {
        const R pm = p[m];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const R d = ldg(DT + (c * NP + m) * NP + n);
          dp[c] += d * pm;
          div += ldg(DV + (c * NP + m) * NP + n) * v[c * NP + m];
        }
      }
      const R* G = sg + e * GEO_PYR;
      acc[s][0] = skew ? div : -div;
#pragma unroll
      for (int x = 0; x < 3; ++x)
        acc[s][1 + x] = -(G[x] * dp[0] + G[3 + x] * dp[1] + G[6 + x] * dp[2]);
    }
  }

  const R pen = R(M.penalty_scale);
  const R* ET = (const R*)T.op[5];
  for (int i = tid; i < ne * NFP; i += NT) {
    const int e = i / NFP, j = i - e * NFP;
    int f, jj;
    if (j < NFQ) { f = 0; jj = j; }
    else { f = 1 + (j - NFQ) / NFN; jj = (j - NFQ) - (f - 1) * NFN; }
    const int k = sk[e];
    const R* qe = sq + e * 4 * NP;
    R own[4] = {R(0), R(0), R(0), R(0)};
    for (int m = 0; m < NP; ++m) {
      const R ev = ldg(ET + m * NFP + j);
#pragma unroll
      for (int c = 0; c < 4; ++c) own[c] += ev * qe[c * NP + m];
    }
    const R um[3] = {own[1], own[2], own[3]};
    const R* g = sg + e * GEO_PYR + 9 + 4 * f;
    const R nrm[3] = {g[0], g[1], g[2]};
    const int code = __ldg(T.nbr_code + (size_t)k * NF_PYR + f);
    const R zm = smat[e * 4 + 2];
    R pp, up[3], zp;
    if (code & HW_NBR_BOUNDARY) {
      pp = -own[0]; up[0] = um[0]; up[1] = um[1]; up[2] = um[2]; zp = zm;
    } else {
      const int k2 = __ldg(T.nbr_elem + (size_t)k * NF_PYR + f);
      R tr[4];
      neighbour_trace<N, R>(M, Q, code, k2, jj, f != 0, tr);
      pp = tr[0]; up[0] = tr[1]; up[1] = tr[2]; up[2] = tr[3];
      zp = neighbour_z<R>(M, code, k2);
    }
    R tp, tu, fp, fu;
    penalties(zm, zp, pen, tp, tu);
    upwind_flux(own[0], um, pp, up, nrm, tp, tu, skew, fp, fu);
    sf[(e * NFP + j) * 2 + 0] = fp * g[3];
    sf[(e * NFP + j) * 2 + 1] = fu * g[3];
  }
  __syncthreads();

  const R* LT = (const R*)T.op[6];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = tid + s * NT;
    const int e = i / NP, n = i - e * NP;
    if (e >= ne) continue;
    const R* fl = sf + e * NFP * 2;
    const R* g = sg + e * GEO_PYR + 9;
    for (int f = 0; f < 5; ++f) {
      const int j0 = f == 0 ? 0 : NFQ + (f - 1) * NFN;
      const int cnt = f == 0 ? NFQ : NFN;
      R tp = R(0), tu = R(0);
      for (int jj = 0; jj < cnt; ++jj) {
        const int j = j0 + jj;
        const R l = ldg(LT + j * NP + n);
        tp += l * fl[2 * j];
        tu += l * fl[2 * j + 1];
      }
      acc[s][0] += tp;
      acc[s][1] += g[4 * f + 0] * tu;
      acc[s][2] += g[4 * f + 1] * tu;
      acc[s][3] += g[4 * f + 2] * tu;
    }
    const R kap = smat[e * 4 + 0], irho = smat[e * 4 + 1];
    const size_t base = (size_t)sk[e] * 4 * NP + n;
    const R* qe = sq + e * 4 * NP + n;
    epilogue<R>(E, HW_PYRAMID, base, acc[s][0] * kap, qe[0]);
#pragma unroll
    for (int c = 1; c < 4; ++c)
      epilogue<R>(E, HW_PYRAMID, base + c * NP, acc[s][c] * irho, qe[c * NP]);
  }
}

// ------------------------------------------------------------------ wedge
// LSC-DG wedge, skew form, affine (hybridwave/dg.py:423-444): two passes
// through the (N+1)^3 cubature points; identity mass; traces carry 1/sqrt(J).
template <int N, typename R>
struct WedgeK {
  using D = Dims<N>;
  static constexpr int NP = D::NP_WEDGE, NQ = D::NQ_WEDGE, NFN = D::NFN, NFQ = D::NFQ,
                       NFP = D::NFP_WEDGE;
  static constexpr int EPB = (NT / NQ) > 0 ? (NT / NQ) : 1;
  static constexpr int S = (EPB * NP + NT - 1) / NT;
  static constexpr int SQ = 0, SW = SQ + EPB * 4 * NP, SF = SW + EPB * 6 * NQ,
                       SG = SF + EPB * NFP * 2, SM = SG + EPB * GEO_WEDGE,
                       SMEM = SM + EPB * 4;
};

template <int N, typename R>
__global__ void __launch_bounds__(NT) wedge_kernel(hw_mesh_t M, hw_fields_t Q, Epi E,
                                                   const int32_t* __restrict__ list,
                                                   int64_t nwork) {
  using K_ = WedgeK<N, R>;
  constexpr int NP = K_::NP, NQ = K_::NQ, NFN = K_::NFN, NFQ = K_::NFQ, NFP = K_::NFP,
                EPB = K_::EPB, S = K_::S;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sm = reinterpret_cast<R*>(smem_raw);
  R* sq = sm + K_::SQ;
  R* sw = sm + K_::SW;
  R* sf = sm + K_::SF;
  R* sg = sm + K_::SG;
  R* smat = sm + K_::SM;
  __shared__ int sk[EPB];

  const hw_type_t& T = M.t[HW_WEDGE];
  const int tid = threadIdx.x;
  const int64_t w0 = (int64_t)blockIdx.x * EPB;
  const int ne = (int)((nwork - w0) < EPB ? (nwork - w0) : EPB);
  if (tid < ne) sk[tid] = list ? list[w0 + tid] : (int)(w0 + tid);
  __syncthreads();

  const R* q = (const R*)Q.p[HW_WEDGE];
  for (int i = tid; i < ne * 4 * NP; i += NT) {
    const int e = i / (4 * NP), r = i - e * 4 * NP;
    sq[i] = ldg(q + (size_t)sk[e] * 4 * NP + r);
  }
  for (int i = tid; i < ne * GEO_WEDGE; i += NT) {
    const int e = i / GEO_WEDGE, r = i - e * GEO_WEDGE;
    sg[i] = ldg((const R*)T.geo + (size_t)sk[e] * GEO_WEDGE + r);
  }
  for (int i = tid; i < ne * 4; i += NT)
    smat[i] = ldg((const R*)T.mat + (size_t)sk[i / 4] * 4 + (i & 3));
  __syncthreads();

  // trial pass at cubature points
  const R* VT = (const R*)T.op[0];    // (NP, NQ)
  const R* D3T = (const R*)T.op[1];   // (3, NP, NQ)
  const R* wq = (const R*)T.op[4];
  for (int i = tid; i < ne * NQ; i += NT) {
    const int e = i / NQ, qi = i - e * NQ;
    const R* qe = sq + e * 4 * NP;
    R U[3] = {R(0), R(0), R(0)}, dp[3] = {R(0), R(0), R(0)};
#pragma unroll 2
    for (int m = 0; m < NP; ++m) {
      const R v = ldg(VT + m * NQ + qi);
      const R pm = qe[m];
      U[0] += v * qe[NP + m];
      U[1] += v * qe[2 * NP + m];
      U[2] += v * qe[3 * NP + m];
#pragma unroll
      for (int c = 0; c < 3; ++c) dp[c] += ldg(D3T + (c * NP + m) * NQ + qi) * pm;
    }
    const R* G = sg + e * GEO_WEDGE;
    const R w = ldg(wq + qi);
    R* o = sw + e * 6 * NQ + qi;
#pragma unroll
    for (int x = 0; x < 3; ++x) o[x * NQ] = w * (G[x] * dp[0] + G[3 + x] * dp[1] + G[6 + x] * dp[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c)
      o[(3 + c) * NQ] = w * (G[c * 3] * U[0] + G[c * 3 + 1] * U[1] + G[c * 3 + 2] * U[2]);
  }
  __syncthreads();

  // test pass
  const R* V = (const R*)T.op[2];     // (NQ, NP)
  const R* D3 = (const R*)T.op[3];    // (3, NQ, NP)
  R acc[S][4];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = tid + s * NT;
    const int e = i / NP, n = i - e * NP;
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[s][c] = R(0);
    if (e < ne) {
      const R* o = sw + e * 6 * NQ;
      R rp = R(0), ru[3] = {R(0), R(0), R(0)};
#pragma unroll 2
      for (int qi = 0; qi < NQ; ++qi) {
        const R v = ldg(V + qi * NP + n);
        ru[0] += v * o[qi];
        ru[1] += v * o[NQ + qi];
        ru[2] += v * o[2 * NQ + qi];
#pragma unroll
        for (int c = 0; c < 3; ++c) rp += ldg(D3 + (c * NQ + qi) * NP + n) * o[(3 + c) * NQ + qi];
      }
      acc[s][0] = rp;
      acc[s][1] = -ru[0];
      acc[s][2] = -ru[1];
      acc[s][3] = -ru[2];
    }
  }

  const R pen = R(M.penalty_scale);
  const R* ET = (const R*)T.op[5];
  for (int i = tid; i < ne * NFP; i += NT) {
    const int e = i / NFP, j = i - e * NFP;
    int f, jj;
    bool tri;
    if (j < 2 * NFN) { f = j / NFN; jj = j - f * NFN; tri = true; }
    else { f = 2 + (j - 2 * NFN) / NFQ; jj = (j - 2 * NFN) - (f - 2) * NFQ; tri = false; }
    const int k = sk[e];
    const R* qe = sq + e * 4 * NP;
    const R isj = sg[e * GEO_WEDGE + 9];
    R own[4] = {R(0), R(0), R(0), R(0)};
    for (int m = 0; m < NP; ++m) {
      const R ev = ldg(ET + m * NFP + j);
#pragma unroll
      for (int c = 0; c < 4; ++c) own[c] += ev * qe[c * NP + m];
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) own[c] *= isj;
    const R um[3] = {own[1], own[2], own[3]};
    const R* g = sg + e * GEO_WEDGE + 10 + 4 * f;
    const R nrm[3] = {g[0], g[1], g[2]};
    const int code = __ldg(T.nbr_code + (size_t)k * NF_WEDGE + f);
    const R zm = smat[e * 4 + 2];
    R pp, up[3], zp;
    if (code & HW_NBR_BOUNDARY) {
      pp = -own[0]; up[0] = um[0]; up[1] = um[1]; up[2] = um[2]; zp = zm;
    } else {
      const int k2 = __ldg(T.nbr_elem + (size_t)k * NF_WEDGE + f);
      R tr[4];
      neighbour_trace<N, R>(M, Q, code, k2, jj, tri, tr);
      pp = tr[0]; up[0] = tr[1]; up[1] = tr[2]; up[2] = tr[3];
      zp = neighbour_z<R>(M, code, k2);
    }
    R tp, tu, fp, fu;
    penalties(zm, zp, pen, tp, tu);
    upwind_flux(own[0], um, pp, up, nrm, tp, tu, true, fp, fu);
    sf[(e * NFP + j) * 2 + 0] = fp * g[3];
    sf[(e * NFP + j) * 2 + 1] = fu * g[3];
  }
  __syncthreads();

  const R* LT = (const R*)T.op[6];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = tid + s * NT;
    const int e = i / NP, n = i - e * NP;
    if (e >= ne) continue;
    const R* fl = sf + e * NFP * 2;
    const R* g = sg + e * GEO_WEDGE + 10;
    for (int f = 0; f < 5; ++f) {
      const int j0 = f < 2 ? f * NFN : 2 * NFN + (f - 2) * NFQ;
      const int cnt = f < 2 ? NFN : NFQ;
      R tp = R(0), tu = R(0);
      for (int jj = 0; jj < cnt; ++jj) {
        const int j = j0 + jj;
        const R l = ldg(LT + j * NP + n);
        tp += l * fl[2 * j];
        tu += l * fl[2 * j + 1];
      }
      acc[s][0] += tp;
      acc[s][1] += g[4 * f + 0] * tu;
      acc[s][2] += g[4 * f + 1] * tu;
      acc[s][3] += g[4 * f + 2] * tu;
    }
    const R kap = smat[e * 4 + 0], irho = smat[e * 4 + 1];
    const size_t base = (size_t)sk[e] * 4 * NP + n;
    const R* qe = sq + e * 4 * NP + n;
    epilogue<R>(E, HW_WEDGE, base, acc[s][0] * kap, qe[0]);
#pragma unroll
    for (int c = 1; c < 4; ++c)
      epilogue<R>(E, HW_WEDGE, base + c * NP, acc[s][c] * irho, qe[c * NP]);
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
  // G = F^{-1}: G[c][x]
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

template <int N, typename R>
struct HexK {
  using D = Dims<N>;
  static constexpr int N1 = D::N1, NP = D::NP_HEX, NFQ = D::NFQ, NFP = D::NFP_HEX;
  static constexpr int EPB = (NT / NP) > 0 ? (NT / NP) : 1;
  static constexpr int S = (EPB * NP + NT - 1) / NT;
  static constexpr int SQ = 0, SF = SQ + EPB * 4 * NP, SG = SF + EPB * NFP * 4,
                       SM = SG + EPB * GEO_HEX, SD = SM + EPB * 4,
                       SMEM = SD + N1 * N1 + 3 * N1 + 2 * N1;
};

template <int N, typename R>
__global__ void __launch_bounds__(NT) hex_kernel(hw_mesh_t M, hw_fields_t Q, Epi E,
                                                 const int32_t* __restrict__ list,
                                                 int64_t nwork) {
  using K_ = HexK<N, R>;
  constexpr int N1 = K_::N1, NP = K_::NP, NFQ = K_::NFQ, NFP = K_::NFP, EPB = K_::EPB,
                S = K_::S;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sm = reinterpret_cast<R*>(smem_raw);
  R* sq = sm + K_::SQ;
  R* sf = sm + K_::SF;
  R* sg = sm + K_::SG;
  R* smat = sm + K_::SM;
  R* sD = sm + K_::SD;           // D1 (N1 x N1)
  R* sx = sD + N1 * N1;          // 1-D nodes
  R* sw1 = sx + N1;              // 1-D weights
  R* sve = sw1 + N1;             // endpoint rows (2 x N1)
  __shared__ int sk[EPB];

  const hw_type_t& T = M.t[HW_HEX];
  const bool sem = M.formulation == HW_SEM;
  const int tid = threadIdx.x;
  const int64_t w0 = (int64_t)blockIdx.x * EPB;
  const int ne = (int)((nwork - w0) < EPB ? (nwork - w0) : EPB);
  if (tid < ne) sk[tid] = list ? list[w0 + tid] : (int)(w0 + tid);
  if (tid < N1 * N1) sD[tid] = ldg((const R*)T.op[0] + tid);
  if (tid < 2 * N1) sve[tid] = ldg((const R*)T.op[1] + tid);
  if (tid < N1) {
    sw1[tid] = ldg((const R*)T.op[2] + tid);
    sx[tid] = ldg((const R*)T.op[4] + tid);
  }
  __syncthreads();

  const R* q = (const R*)Q.p[HW_HEX];
  for (int i = tid; i < ne * 4 * NP; i += NT) {
    const int e = i / (4 * NP), r = i - e * 4 * NP;
    sq[i] = ldg(q + (size_t)sk[e] * 4 * NP + r);
  }
  for (int i = tid; i < ne * GEO_HEX; i += NT) {
    const int e = i / GEO_HEX, r = i - e * GEO_HEX;
    sg[i] = ldg((const R*)T.geo + (size_t)sk[e] * GEO_HEX + r);
  }
  for (int i = tid; i < ne * 4; i += NT)
    smat[i] = ldg((const R*)T.mat + (size_t)sk[i / 4] * 4 + (i & 3));
  __syncthreads();

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
      const R J = hex_metric<R>(sg + e * GEO_HEX, sx[ii], sx[jj], sx[kk], G);
      R div = R(0);
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        acc[s][1 + x] = -(G[x] * d[0][0] + G[3 + x] * d[0][1] + G[6 + x] * d[0][2]);
        div += G[x] * d[1 + x][0] + G[3 + x] * d[1 + x][1] + G[6 + x] * d[1 + x][2];
      }
      acc[s][0] = -div;
      minv[s] = R(1) / (sw1[ii] * sw1[jj] * sw1[kk] * J);
    }
  }

  const R pen = R(M.penalty_scale);
  for (int i = tid; i < ne * NFP; i += NT) {
    const int e = i / NFP, j = i - e * NFP;
    const int f = j / NFQ, jj = j - f * NFQ;
    const int k = sk[e];
    const int* tab = T.iop[0] + 3 * j;
    const int base = __ldg(tab), stride = __ldg(tab + 1), end = __ldg(tab + 2);
    const R* qe = sq + e * 4 * NP;
    R own[4];
    if (sem) {
      const int node = base + (end ? N : 0) * stride;
#pragma unroll
      for (int c = 0; c < 4; ++c) own[c] = qe[c * NP + node];
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) own[c] = R(0);
#pragma unroll
      for (int l = 0; l < N1; ++l) {
        const R w = sve[end * N1 + l];
#pragma unroll
        for (int c = 0; c < 4; ++c) own[c] += w * qe[c * NP + base + l * stride];
      }
    }
    // face geometry at (xi, eta) = (x[a], x[b]) from the 4 face vertices
    const int a = jj / N1, b = jj - a * N1;
    const R xi = sx[a], eta = sx[b];
    const R* X = sg + e * GEO_HEX;
    R t1[3], t2[3];
    {
      const R g1[4] = {-(R(1) - eta), (R(1) - eta), (R(1) + eta), -(R(1) + eta)};
      const R g2[4] = {-(R(1) - xi), -(R(1) + xi), (R(1) + xi), (R(1) - xi)};
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        R s1 = R(0), s2 = R(0);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const R xv = X[c_hex_face_verts[f][v] * 3 + x];
          s1 += g1[v] * xv;
          s2 += g2[v] * xv;
        }
        t1[x] = R(0.25) * s1;
        t2[x] = R(0.25) * s2;
      }
    }
    R nv[3] = {t1[1] * t2[2] - t1[2] * t2[1], t1[2] * t2[0] - t1[0] * t2[2],
               t1[0] * t2[1] - t1[1] * t2[0]};
    const R Js = sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
    const R nrm[3] = {nv[0] / Js, nv[1] / Js, nv[2] / Js};
    const R wJs = sw1[a] * sw1[b] * Js;
    const R um[3] = {own[1], own[2], own[3]};
    const int code = __ldg(T.nbr_code + (size_t)k * NF_HEX + f);
    const R zm = smat[e * 4 + 2];
    R pp, up[3], zp;
    if (code & HW_NBR_BOUNDARY) {
      pp = -own[0]; up[0] = um[0]; up[1] = um[1]; up[2] = um[2]; zp = zm;
    } else {
      const int k2 = __ldg(T.nbr_elem + (size_t)k * NF_HEX + f);
      R tr[4];
      neighbour_trace<N, R>(M, Q, code, k2, jj, false, tr);
      pp = tr[0]; up[0] = tr[1]; up[1] = tr[2]; up[2] = tr[3];
      zp = neighbour_z<R>(M, code, k2);
    }
    R tp, tu, fp, fu;
    penalties(zm, zp, pen, tp, tu);
    upwind_flux(own[0], um, pp, up, nrm, tp, tu, T.form == HW_FORM_SKEW, fp, fu);
    R* o = sf + (e * NFP + j) * 4;
    o[0] = fp * wJs;
    o[1] = nrm[0] * fu * wJs;
    o[2] = nrm[1] * fu * wJs;
    o[3] = nrm[2] * fu * wJs;
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
      const int pt = __ldg(T.iop[1] + f * NP + n);
      const R* o = fl + (f * NFQ + pt) * 4;
#pragma unroll
      for (int c = 0; c < 4; ++c) lift[c] += w * o[c];
    }
    // only the surface term carries the mass inverse 1/(w3 J): the volume
    // term above is already the cancelled form -grad p, -div u
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[s][c] += lift[c] * minv[s];
    const R kap = smat[e * 4 + 0], irho = smat[e * 4 + 1];
    const size_t base = (size_t)sk[e] * 4 * NP + n;
    const R* qe = sq + e * 4 * NP + n;
    epilogue<R>(E, HW_HEX, base, acc[s][0] * kap, qe[0]);
#pragma unroll
    for (int c = 1; c < 4; ++c)
      epilogue<R>(E, HW_HEX, base + c * NP, acc[s][c] * irho, qe[c * NP]);
  }
}

}  // namespace hw
