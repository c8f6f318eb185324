// Tet RHS + update with the dense contractions on the fp64 tensor cores
// (mma.sync.m8n8k4.f64, SASS DMMA); state storage fp64 or fp32, arithmetic
// fp64 (fp32 storage rounds once, at the store).
//
// A block owns E tets; warp w owns one 8x8 output tile (row tile = 8 nodes,
// column tile = 8 elements).  All per-element smem arrays are element-major
// with an element stride = 4 (mod 16) doubles, so a B-fragment load (4
// consecutive k x 8 elements) touches every bank exactly twice (the minimum
// for 256 B) while whole element rows can be copied with 16-byte cp.async.
//   volume  DP_c = D_c p,  DIV = sum_c D_c v_c          (strong form)
//   lift    P += LIFT_f fp_f,  TU_f = LIFT_f fu_f,  U_x += n_f,x TU_f
// Neighbour face values come through a host-precomputed gather index in
// this element's face-point order (tet_gather_index in device.py) straight
// into registers: loaded before the volume GEMMs, consumed by the flux
// (the kernel is bound by the SM's L1/shared data pipe; a smem staging
// round trip costs more wavefronts than it saves).  Operator fragments are
// stored in A-fragment order (device.mma_fragments): one contiguous 256-byte
// read per fragment.  On B200 DMMA and DFMA have the same peak (37 vs 34
// TF/s measured); DMMA wins by needing 2 operand loads per 256 FMAs.
// Reference arithmetic: hybridwave/dg.py:401-421 (volume), 326-354 (flux),
// 479-490 (mass inverse).
#pragma once
#include "hw_kernels.cuh"

namespace hw {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__host__ __device__ constexpr int stride4mod16(int n) {   // smallest s >= n, s = 4 (mod 16)
  return n + ((4 - n % 16) + 16) % 16;
}

// element stride (in storage scalars) that makes a B-fragment load (4
// consecutive k x 8 elements) conflict-free: fp64 4 (mod 16) doubles, fp32
// 4 (mod 8) floats (one 128-byte wavefront); both keep 16-byte row alignment
template <typename S>
__host__ __device__ constexpr int frag_stride(int n) {
  return sizeof(S) == 8 ? stride4mod16(n) : n + ((4 - n % 8) + 8) % 8;
}

// elements per block (tuning: HW_TET_E2 / HW_TET_E4 for N = 2 / 4)
#ifndef HW_TET_E1
#define HW_TET_E1 32
#endif
#ifndef HW_TET_E2
#define HW_TET_E2 16
#endif
#ifndef HW_TET_E4
#define HW_TET_E4 8
#endif
#ifndef HW_TET_MINB
#define HW_TET_MINB 6
#endif
#ifndef HW_TET_MINB_XW
#define HW_TET_MINB_XW 7
#endif
#ifndef HW_TET_MINB32
#define HW_TET_MINB32 12
#endif

// S: storage type of the state, records and smem (double or float); the
// arithmetic is fp64 throughout (DMMA), fp32 storage rounds at the store
template <int N, typename S = double>
struct TetMma {
  using D = Dims<N>;
  static constexpr int NP = D::NP_TET, NFN = D::NFN, NFP = 4 * D::NFN;
  static constexpr int E = (N == 1) ? HW_TET_E1 : (N == 2 ? HW_TET_E2 : (N == 4 ? HW_TET_E4 : 8));
  static constexpr int CT = E / 8;
  static constexpr int RT = (NP + 7) / 8;
  static constexpr int NPK = ((NP + 3) / 4) * 4;
  static constexpr int NFK = ((NFN + 3) / 4) * 4;
  static constexpr int W = RT * CT;
#ifndef HW_TET_XW
#define HW_TET_XW 1
#endif
  // XW extra warps join the copy / flux phases only (GEMM warps: W).
  // Measured (hybrid:38): fp64 N=3 tet 188.5 -> 180.4 us with one extra warp
  // (MINB 7); slower for fp32 N=3 (141 -> 148) and fp64 N=1,2,4,5.
  static constexpr int XW = (sizeof(S) == 8 && N == 3) ? HW_TET_XW : 0;
  static constexpr int NTH = 32 * (W + XW);
  // q / res rows are contiguous in smem (field stride NP, as in HBM); the
  // K padding of the p-field B fragments reads the next field's values,
  // which the zero-padded A fragments cancel
  static constexpr bool VEC = (4 * NP * sizeof(S)) % 16 == 0;  // 16-byte rows
  static constexpr int EQ = frag_stride<S>(4 * NPK);        // q / res element stride
  static constexpr int EV = frag_stride<S>(3 * NPK);        // v_c
  static constexpr int EF = frag_stride<S>(4 * NFK);        // fp / fu
  // buffers live in disjoint phases share storage: v_c (volume) with fp/fu
  // (flux, lift)
  static constexpr int RA = cmax(EV, 2 * EF);
  static constexpr int SQ = 0, SV = SQ + E * EQ, SFP = SV, SFU = SFP + E * EF,
                       SRES = SV + E * RA, SG = SRES + E * EQ,
                       SMAT = SG + E * GEO_TET, TOTAL = SMAT + E * 4;
  // int region: element ids, own face-node table, then (16-byte aligned)
  // the block's gather-index rows when they arrive by TMA
  static constexpr int SIDX = ((E + NFP + 3) / 4) * 4;
  static constexpr size_t BYTES = sizeof(S) * TOTAL + sizeof(int) * (SIDX + E * NFP);
  // TMA (cp.async.bulk) staging of whole element rows: rows contiguous in
  // smem (no K padding) and every copy a multiple of 16 bytes at 16-byte
  // aligned addresses; otherwise the cp.async path stages them
  static constexpr bool TMA_OK =
      (4 * NP * sizeof(S)) % 16 == 0 && (EQ * sizeof(S)) % 16 == 0 &&
      (SRES * sizeof(S)) % 16 == 0 && (SG * sizeof(S)) % 16 == 0 &&
      (SMAT * sizeof(S)) % 16 == 0 && (TOTAL * sizeof(S)) % 16 == 0 &&
      (E * GEO_TET * sizeof(S)) % 16 == 0 && (E * 4 * sizeof(S)) % 16 == 0 &&
      (NFP * 4) % 16 == 0;
#ifndef HW_TET_MINB_MID
#define HW_TET_MINB_MID 4
#endif
  static constexpr int MINB = (W <= 4) ? (sizeof(S) == 8 ? (XW ? HW_TET_MINB_XW : HW_TET_MINB) : HW_TET_MINB32)
                                       : ((W <= 8) ? HW_TET_MINB_MID : 1);
  // flux items (element, face point) per thread
  static constexpr int IT = (E * NFP + NTH - 1) / NTH;
};

// element rows (K, 4, NP) -> smem [e][field (stride NP)][node]
template <typename L, typename S>
__device__ __forceinline__ void tet_rows(S* dst, const S* src, const int* sk, int ne) {
  constexpr int NP = L::NP, NPK = L::NPK;
  if (L::VEC) {
    copy_rows16<4 * NP, L::EQ, L::NTH, L::E>(dst, src, sk, ne);
  } else {
    for (int i = threadIdx.x; i < ne * 4 * NP; i += L::NTH) {
      const int e = i / (4 * NP), r = i - e * 4 * NP;
      const int fld = r / NP, n = r - fld * NP;
      cp_async(dst + e * L::EQ + fld * NP + n, src + (size_t)sk[e] * 4 * NP + r);
    }
  }
}

// MMA column c of a column tile holds element pi(c) of its 8: swapping the
// elements 4<->5 and 6<->7 makes the accumulator layout (lane holds columns
// 2(lane&3) + {0,1}) touch four different bank groups in the epilogue
// (elements {0,2,5,7} and {1,3,4,6} instead of {0,2,4,6}); B-fragment loads
// stay conflict-free under any column permutation.
__device__ __forceinline__ int tet_col_elem(int c) { return c ^ ((c >> 2) & 1); }

// SK: skew form (forms_override testing hook) as a compile-time variant so
// the production strong-form kernel carries none of its code
template <int N, typename S, bool SK = false>
__global__ void __launch_bounds__(TetMma<N, S>::NTH, TetMma<N, S>::MINB)
    tet_mma_kernel(hw_mesh_t M, hw_fields_t Q, Epi E, const int32_t* __restrict__ list,
                   int64_t nwork) {
  using L = TetMma<N, S>;
  using R = double;   // arithmetic
  constexpr int NP = L::NP, NFN = L::NFN, NFP = L::NFP, EB = L::E, NPK = L::NPK,
                NFK = L::NFK, NTH = L::NTH, EQ = L::EQ, EV = L::EV, EF = L::EF, IT = L::IT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S* sm = reinterpret_cast<S*>(smem_raw);
  int* sk = reinterpret_cast<int*>(sm + L::TOTAL);
  int* sfn = sk + EB;               // own face node table
  S* sq = sm + L::SQ;
  S* sres = sm + L::SRES;
  S* sv = sm + L::SV;
  S* sfp = sm + L::SFP;
  S* sfu = sm + L::SFU;
  S* sg = sm + L::SG;
  S* smat = sm + L::SMAT;

  const hw_type_t& TY = M.t[HW_TET];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t w0 = (int64_t)blockIdx.x * EB;
  const int ne = (int)((nwork - w0) < EB ? (nwork - w0) : EB);
  const bool lsrk = E.mode == MODE_LSRK;

  // TMA path: a full block of consecutive elements (no subset list)
  __shared__ __align__(8) uint64_t tbar[2];
  const bool tma = L::TMA_OK && list == nullptr && ne == EB;
  int* sidx = reinterpret_cast<int*>(sm + L::TOTAL) + L::SIDX;
  const S* q = (const S*)Q.p[HW_TET];
  if (tma && tid == 0) {
    mbar_init(&tbar[0], 1);
    mbar_init(&tbar[1], 1);
    mbar_fence_init();
  }
  if (tid < EB) sk[tid] = tid < ne ? (list ? list[w0 + tid] : (int)(w0 + tid)) : 0;
  for (int i = tid; i < NFP; i += NTH) sfn[i] = __ldg(TY.iop[0] + i);
  // K padding must be zero for the DMMA (rows are never written by copies)
  constexpr int PADN = (NPK > NP) ? NPK - NP : 1, PADF = (NFK > NFN) ? NFK - NFN : 1;
  if (NPK > NP)   // v_c K padding, and the q-row tail the last field's padding reads
    for (int i = tid; i < EB * 4 * PADN; i += NTH) {
      const int e = i / (4 * PADN), r = i - e * 4 * PADN;
      const int fld = r / PADN, n = NP + r - fld * PADN;
      if (fld == 0) sq[e * EQ + 3 * NP + n] = S(0);
      else sv[e * EV + (fld - 1) * NPK + n] = S(0);
    }
  __syncthreads();

  // ---- P0: element rows, records and the gather index.  TMA path: warp 0
  // issues one bulk copy per element row (q; the LSRK residual on a second
  // barrier, waited for only by the epilogue) and one per record array.
  // cp.async path (subset lists, partial blocks, padded rows): per-thread
  // 16-byte copies and the gather index straight into registers.
  // Thread-item u is (e, j) = (tid + u * NTH) / NFP, % NFP, the mapping the
  // flux loop uses.
  constexpr unsigned ROWB = 4 * NP * sizeof(S);
  int gv[IT];
  if (tma) {
    if (warp == 0) {
      if (lane == 0) {
        mbar_expect_tx(&tbar[0], EB * ROWB + EB * (GEO_TET + 4) * sizeof(S) + EB * NFP * 4);
        if (lsrk) mbar_expect_tx(&tbar[1], EB * ROWB);
      }
      __syncwarp();
      const S* res = (const S*)E.res[HW_TET];
      for (int e = lane; e < EB; e += 32) {
        bulk_load(sq + e * EQ, q + (size_t)(w0 + e) * 4 * NP, ROWB, &tbar[0]);
        if (lsrk) bulk_load(sres + e * EQ, res + (size_t)(w0 + e) * 4 * NP, ROWB, &tbar[1]);
      }
      if (lane == 0) {
        bulk_load(sg, (const S*)TY.geo + (size_t)w0 * GEO_TET, EB * GEO_TET * sizeof(S),
                  &tbar[0]);
        bulk_load(smat, (const S*)TY.mat + (size_t)w0 * 4, EB * 4 * sizeof(S), &tbar[0]);
        bulk_load(sidx, TY.iop[1] + (size_t)w0 * NFP, EB * NFP * 4, &tbar[0]);
      }
    }
    mbar_wait(&tbar[0], 0);
#pragma unroll
    for (int u = 0; u < IT; ++u) {
      const int i = tid + u * NTH;
      gv[u] = i < EB * NFP ? sidx[i] : -1;
    }
  } else {
    tet_rows<L>(sq, q, sk, ne);
    copy_rows<GEO_TET, GEO_TET, NTH, EB>(sg, (const S*)TY.geo, sk, ne);
    copy_rows<4, 4, NTH, EB>(smat, (const S*)TY.mat, sk, ne);
#pragma unroll
    for (int u = 0; u < IT; ++u) {
      const int i = tid + u * NTH;
      gv[u] = -1;
      if (i < ne * NFP) gv[u] = __ldg(TY.iop[1] + (size_t)sk[i / NFP] * NFP + i % NFP);
    }
    cp_async_commit();
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
  }

  // ---- P1: neighbour face-node values (registers, consumed by the flux)
  R nb[IT][4];
#pragma unroll
  for (int u = 0; u < IT; ++u) {
    const int g = gv[u];
    if (g >= 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) nb[u][c] = R(ldg(q + (size_t)g + c * NP));
    } else if (g != -1) {   // pyramid / wedge neighbour: its published face trace
      const unsigned v = (unsigned)(-3 - g);
      const int t2 = (v & 1u) ? HW_WEDGE : HW_PYRAMID;
      const int nfp2 = (v & 1u) ? Dims<N>::NFP_WEDGE : Dims<N>::NFP_PYR;
      const S* src = (const S*)M.tr_in[t2] + (size_t)(v >> 1);
#pragma unroll
      for (int c = 0; c < 4; ++c) nb[u][c] = R(ldg(src + c * nfp2));
    }
  }

  // v_c = sum_x G[c][x] u_x
  for (int i = tid; i < ne * NP; i += NTH) {
    const int e = i / NP, n = i - e * NP;
    const S* G = sg + e * GEO_TET;
    const S* u = sq + e * EQ + n;
    const R u0 = u[NP], u1 = u[2 * NP], u2 = u[3 * NP];
#pragma unroll
    for (int c = 0; c < 3; ++c)
      sv[e * EV + c * NPK + n] = S(R(G[c * 3]) * u0 + R(G[c * 3 + 1]) * u1 + R(G[c * 3 + 2]) * u2);
  }
  __syncthreads();

  // ---- P2: volume GEMMs on DMMA
  const int rt = warp / L::CT, ct = warp - rt * L::CT;
  const int bk = lane & 3, bcol = ct * 8 + tet_col_elem(lane >> 2);
  constexpr bool skew = SK;
  R dp[3][2] = {{0, 0}, {0, 0}, {0, 0}}, dv[2] = {0, 0};
  const bool gw = warp < L::W;   // GEMM warp
  if (gw) {
    const R* Dg = (const R*)TY.op[2];   // [3][RT][NPK/4][32] A fragments, zero padded
    const R* Bg = (const R*)TY.op[5];   // skew: invM D_c^T M fragments
    const S* bq = sq + bcol * EQ + bk;
    const S* bv = sv + bcol * EV + bk;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
      for (int ks = 0; ks < NPK / 4; ++ks) {
        const int fi = (((c * L::RT + rt) * (NPK / 4) + ks) << 5) + lane;
        const R a = ldg(Dg + fi);
        dmma884(dp[c][0], dp[c][1], a, bq[ks * 4]);
        dmma884(dv[0], dv[1], skew ? ldg(Bg + fi) : a, bv[c * NPK + ks * 4]);
      }
    }
  }
  __syncthreads();

  // ---- P3: flux at the face nodes (face point fastest across threads)
  if (NFK > NFN)      // K padding of fp/fu (their storage held v_c until now)
    for (int i = tid; i < EB * 8 * PADF; i += NTH) {
      const int e = i / (8 * PADF), r = i - e * 8 * PADF;
      const int fld = r / PADF, n = NFN + r - fld * PADF;
      (fld < 4 ? sfp : sfu)[e * EF + (fld & 3) * NFK + n] = S(0);
    }
  const R pen = R(M.penalty_scale);
#pragma unroll
  for (int u = 0; u < IT; ++u) {
    const int i = tid + u * NTH;
    if (i >= ne * NFP) break;
    const int e = i / NFP, j = i - e * NFP;
    const int f = j / NFN, jj = j - f * NFN;
    const int node = sfn[j];
    const S* qe = sq + e * EQ + node;
    const R pm = qe[0];
    const R um[3] = {qe[NP], qe[2 * NP], qe[3 * NP]};
    const S* g = sg + e * GEO_TET + 9 + FS * f;
    const R nrm[3] = {g[0], g[1], g[2]};
    R pp, up[3];
    if (gv[u] != -1) {
      pp = nb[u][0]; up[0] = nb[u][1]; up[1] = nb[u][2]; up[2] = nb[u][3];
    } else {   // boundary mirror p+ = -p-, u+ = u-
      pp = -pm; up[0] = um[0]; up[1] = um[1]; up[2] = um[2];
    }
    R tp, tu, fp, fu;
    penalties(R(g[4]), R(g[5]), pen, tp, tu);
    upwind_flux(pm, um, pp, up, nrm, tp, tu, skew, fp, fu);
    sfp[e * EF + f * NFK + jj] = S(fp * R(g[3]));
    sfu[e * EF + f * NFK + jj] = S(fu * R(g[3]));
  }
  __syncthreads();
  // LSRK residual rows, fetched behind the lift GEMM (the TMA path issued
  // them with the other rows)
  if (lsrk && !tma) {
    tet_rows<L>(sres, (const S*)E.res[HW_TET], sk, ne);
    cp_async_commit();
  }

  // ---- P4: lift on DMMA, combine, epilogue
  int ecol[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) ecol[i] = ct * 8 + tet_col_elem((lane & 3) * 2 + i);
  R accp[2] = {skew ? dv[0] : -dv[0], skew ? dv[1] : -dv[1]};
  R accu[3][2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const S* G = sg + ecol[i] * GEO_TET;
#pragma unroll
    for (int x = 0; x < 3; ++x)
      accu[x][i] = -(R(G[x]) * dp[0][i] + R(G[3 + x]) * dp[1][i] + R(G[6 + x]) * dp[2][i]);
  }
  if (gw) {
    const R* Lg = (const R*)TY.op[3];   // [4][RT][NFK/4][32] A fragments
    const S* bp = sfp + bcol * EF + bk;
    const S* bu = sfu + bcol * EF + bk;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      R tu[2] = {0, 0};
#pragma unroll
      for (int ks = 0; ks < NFK / 4; ++ks) {
        const R a = ldg(Lg + (((f * L::RT + rt) * (NFK / 4) + ks) << 5) + lane);
        dmma884(accp[0], accp[1], a, bp[f * NFK + ks * 4]);
        dmma884(tu[0], tu[1], a, bu[f * NFK + ks * 4]);
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const S* g = sg + ecol[i] * GEO_TET + 9 + FS * f;
        accu[0][i] += R(g[0]) * tu[i];
        accu[1][i] += R(g[1]) * tu[i];
        accu[2][i] += R(g[2]) * tu[i];
      }
    }
  }
  const int n = rt * 8 + (lane >> 2);
  if (tma) {
    // results into the staged rows (each (node, element) is read and
    // written by one lane only), then one bulk store per element row
    if (lsrk) mbar_wait(&tbar[1], 0);
    if (gw && n < NP) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int e = ecol[i];
        const S kap = smat[e * 4 + 0], irho = smat[e * 4 + 1];
        S* qe = sq + e * EQ + n;
        S* re = sres + e * EQ + n;
        const size_t base = (size_t)(w0 + e) * 4 * NP + n;
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const S v = (x == 0 ? S(accp[i] * R(kap)) : S(accu[x - 1][i] * R(irho))) +
                      frc_at<S>(E, HW_TET, base + x * NP);
          const S qv = qe[x * NP];
          if (lsrk) {
            const S r = S(E.a) * re[x * NP] + S(E.dt) * v;
            re[x * NP] = r;
            qe[x * NP] = qv + S(E.b) * r;
          } else if (E.mode == MODE_RHS) {
            qe[x * NP] = v;
          } else {
            S acc = S(E.c0) * v;
            if (E.nhist > 1) acc += S(E.c1) * ((const S*)E.h1[HW_TET])[base + x * NP];
            if (E.nhist > 2) acc += S(E.c2) * ((const S*)E.h2[HW_TET])[base + x * NP];
            re[x * NP] = v;
            qe[x * NP] = qv + S(E.dt) * acc;
          }
        }
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (warp == 0) {
      S* d1 = (S*)(E.mode == MODE_RHS ? E.out[HW_TET] : E.qout[HW_TET]);
      S* d2 = (S*)(lsrk ? E.res[HW_TET] : (E.mode == MODE_AB ? E.out[HW_TET] : nullptr));
      for (int e = lane; e < EB; e += 32) {
        bulk_store(d1 + (size_t)(w0 + e) * 4 * NP, sq + e * EQ, ROWB);
        if (d2) bulk_store(d2 + (size_t)(w0 + e) * 4 * NP, sres + e * EQ, ROWB);
      }
      bulk_commit();
      bulk_wait_read();
    }
    return;
  }
  if (lsrk) {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
  }
  if (gw && n < NP) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int e = ecol[i];
      if (e >= ne) continue;
      const R kap = smat[e * 4 + 0], irho = smat[e * 4 + 1];
      const size_t base = (size_t)sk[e] * 4 * NP + n;
      const S* qe = sq + e * EQ + n;
      const S* re = sres + e * EQ + n;
      epilogue_s<S>(E, HW_TET, base, S(accp[i] * kap) + frc_at<S>(E, HW_TET, base), qe[0],
                    re[0]);
#pragma unroll
      for (int x = 0; x < 3; ++x)
        epilogue_s<S>(E, HW_TET, base + (1 + x) * NP,
                      S(accu[x][i] * irho) + frc_at<S>(E, HW_TET, base + (1 + x) * NP),
                      qe[(1 + x) * NP],
                      re[(1 + x) * NP]);
    }
  }
}

}  // namespace hw
