// Wedge / pyramid RHS + update with the dense contractions on the fp64
// tensor cores (mma.sync.m8n8k4.f64); storage fp64 or fp32, arithmetic fp64.  Same organisation as
// tet_mma_kernel; in addition these types publish the face traces of their
// new state (trace buffer, see hw_kernels.cuh) with a third GEMM
//   TR = E q_out    (face points x (element, field)),
// and read their own traces of the input state from the trace buffer.
//   volume  DP_c = A_c p;  DIV = sum_c A_c v_c (strong) | sum_c A_c^T v_c (skew)
//   lift    P += LIFT_f fp_f,  TU_f = LIFT_f fu_f,  U_x += n_f,x TU_f
// A_c = D_c (pyramid), S_c = V^T W D3_c (affine wedge); reference
// arithmetic hybridwave/dg.py:423-463, 326-354, 479-490.
#pragma once
#include "hw_tet_mma.cuh"

namespace hw {

// S: storage type (double or float); arithmetic fp64 (DMMA) throughout
template <int N, int T, typename S = double>
struct DMma {
  using X = TT<N, T>;
  using D = Dims<N>;
  static constexpr int NP = X::NP, NF = X::NF, NFP = X::NFP, GEO = X::GEO, GF = X::GF;
  static constexpr int E = 8;
  static constexpr int RT = (NP + 7) / 8;
  static constexpr int RT8 = RT * 8;
  static constexpr int NPK = ((NP + 3) / 4) * 4;
  // small RT: two warp groups of RT warps, group 0 grad p + the u lift
  // (u rows), group 1 div v + the p lift (p rows); large RT (N >= 4): one
  // warp per row tile does both (keeps the block at <= RT warps)
#ifndef HW_DENSE_SPLIT_MAX_RT
#define HW_DENSE_SPLIT_MAX_RT 6
#endif
  static constexpr bool SPLIT = RT <= HW_DENSE_SPLIT_MAX_RT;
  static constexpr int W = SPLIT ? 2 * RT : RT;
  static constexpr int NTH = 32 * W;
  __host__ __device__ static constexpr int kf(int f) { return ((X::cnt(f) + 3) / 4) * 4; }
  __host__ __device__ static constexpr int koff(int f) {
    int s = 0;
    for (int g = 0; g < f; ++g) s += kf(g);
    return s;
  }
  static constexpr int NFKT = koff(NF);                 // padded, face-concatenated K of the lift
  // koff for a runtime face index: select chain (the constexpr loop would
  // become a runtime loop)
  __device__ __forceinline__ static int koff_rt(int f) {
    int o = 0;
#pragma unroll
    for (int g = 0; g < NF - 1; ++g) o += (g < f) ? kf(g) : 0;
    return o;
  }
  // operand fragments are stored in k-step pairs (16-byte loads)
  static constexpr int KSP = NPK / 4, KPP = (KSP + 1) / 2;         // volume / trace GEMMs
  static constexpr int KSL = NFKT / 4, KPL = (KSL + 1) / 2;        // lift
  __host__ __device__ static constexpr int kface(int j) {          // face of lift k-step j
    int f = 0;
    for (int g = 1; g < NF; ++g)
      if (4 * j >= koff(g)) f = g;
    return f;
  }
  static constexpr int RTF = (NFP + 7) / 8;             // row tiles of the trace GEMM
  static constexpr int GEOS = GEO | 1;   // odd smem stride: per-element record reads spread over banks
  // q / res field stride: the trace GEMM's B fragments (8 columns = 2
  // elements x 4 fields) conflict-free: fp64 4 or 12 (mod 16) doubles,
  // fp32 8 or 24 (mod 32) floats
  __host__ __device__ static constexpr int qf_stride(int n) {
    if (sizeof(S) == 8)
      return n + ((n % 16 <= 4) ? 4 - n % 16 : (n % 16 <= 12 ? 12 - n % 16 : 20 - n % 16));
    return n + ((n % 32 <= 8) ? 8 - n % 32 : (n % 32 <= 24 ? 24 - n % 32 : 40 - n % 32));
  }
  static constexpr int QF = qf_stride(NPK);
  static constexpr int EQ = frag_stride<S>(4 * QF);
  static constexpr int EV = frag_stride<S>(3 * NPK);
  static constexpr int EF = frag_stride<S>(NFKT);
  // own traces [4][NFP] in my face-point order (stride padded by 16 bytes:
  // 16-byte copies); neighbour values are gathered into registers
  static constexpr int V16 = 16 / sizeof(S);
  static constexpr int ETR = 4 * NFP + V16;
  // storage shared by phase-disjoint buffers: v_c (volume) with fp/fu
  // (flux, lift); own traces (flux) with the residual (epilogue)
  static constexpr int RA = cmax(EV, 2 * EF), RB = cmax(ETR, EQ);
  static constexpr int SQ = 0, SV = SQ + E * EQ, SFP = SV, SFU = SFP + E * EF,
                       STR = SV + E * RA, SRES = STR,
                       SG = STR + E * RB, SMAT = SG + E * GEOS, TOTAL = SMAT + E * 4;
  static constexpr size_t BYTES = sizeof(S) * TOTAL + sizeof(int) * (E + E * NF);
  // blocks per SM the register allocation targets (split layouts; the
  // large-RT layouts use the compiler's default heuristic, see
  // dense_mma_kernel_big: an explicit 1 would let it take 150+ registers)
#ifndef HW_DENSE_MINB
#define HW_DENSE_MINB 3
#endif
#ifndef HW_DENSE_MINB32
#define HW_DENSE_MINB32 5
#endif
  static constexpr int MINB = sizeof(S) == 8 ? HW_DENSE_MINB : HW_DENSE_MINB32;
  static constexpr int BIG_MINB = (65536 / (NTH * 64)) > 1 ? 65536 / (NTH * 64) : 1;
};

// element rows (K, 4, NP) -> smem [e][field (stride QF)][node]
template <typename L, typename S>
__device__ __forceinline__ void copy_q_rows(S* dst, const S* src, const int* sk, int ne) {
  constexpr int NP = L::NP, V = L::V16;
  if (NP % V == 0) {
    // warp per element: sk and the bases are warp-uniform
    constexpr int CF = NP / V, CH = 4 * CF;   // 16-byte chunks per field / element
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int e = warp; e < ne; e += L::W) {
      const S* s = src + (size_t)sk[e] * 4 * NP;
      S* d = dst + e * L::EQ;
#pragma unroll
      for (int c0 = 0; c0 < CH; c0 += 32) {
        const int r = c0 + lane;
        if (r < CH) {
          const int fld = r / CF, c = r - fld * CF;
          cp_async16(d + fld * L::QF + V * c, s + fld * NP + V * c);
        }
      }
    }
  } else {
    for (int i = threadIdx.x; i < ne * 4 * NP; i += L::NTH) {
      const int e = i / (4 * NP), r = i - e * 4 * NP, fld = r / NP, n = r - fld * NP;
      cp_async(dst + e * L::EQ + fld * L::QF + n, src + (size_t)sk[e] * 4 * NP + r);
    }
  }
}

// TR = E q for the block's elements, q in smem ([e][field (stride QF)]
// [node], K padding zero): DMMA with the element-field pairs as columns (4
// column tiles for E = 8), one row tile of face points per warp pass, each
// A fragment feeding 4 MMAs.  Wedges scale by 1/sqrt(J) (record word 9).
template <typename L, int T, typename S>
__device__ __forceinline__ void publish_mma(const hw_type_t& TY, const S* sq, const S* sg,
                                            const int* sk, int ne, S* tro) {
  using R = double;
  constexpr int NFP = L::NFP;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int er = lane >> 2, bk = lane & 3;
  const R* Ep = (const R*)TY.op[7];   // [RTF][NPK/4][32] trace-operator fragments
  for (int rf = warp; rf < L::RTF; rf += L::W) {
    R y[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    const R* arow_p = Ep + ((rf * L::KPP) << 6) + 2 * lane;
    double2 pr;
#pragma unroll
    for (int ks = 0; ks < L::KSP; ++ks) {
      if (!(ks & 1)) pr = ldg2(arow_p + ((ks >> 1) << 6));
      const R a = (ks & 1) ? pr.y : pr.x;
#pragma unroll
      for (int cf = 0; cf < 4; ++cf) {
        const int col = cf * 8 + er;
        dmma884(y[cf][0], y[cf][1], a, sq[(col >> 2) * L::EQ + (col & 3) * L::QF + bk + ks * 4]);
      }
    }
    const int j = rf * 8 + er;
    if (j < NFP) {
#pragma unroll
      for (int cf = 0; cf < 4; ++cf) {
        const int c0 = cf * 8 + (lane & 3) * 2;      // output columns c0, c0+1
        const int e = c0 >> 2;
        if (e >= ne) continue;
        R s = R(1);
        if (T == HW_WEDGE) s = R(sg[e * L::GEOS + 9]);
        S* o = tro + (size_t)sk[e] * 4 * NFP + j;
        o[(c0 & 3) * NFP] = S(y[cf][0] * s);
        o[((c0 & 3) + 1) * NFP] = S(y[cf][1] * s);
      }
    }
  }
}

template <int N, int T, typename S>
__device__ __forceinline__ void dense_mma_body(const hw_mesh_t& M, const hw_fields_t& Q,
                                               const Epi& E, const int32_t* __restrict__ list,
                                               int64_t nwork) {
  using L = DMma<N, T, S>;
  using X = TT<N, T>;
  using R = double;
  constexpr int NP = L::NP, NF = L::NF, NFP = L::NFP, EB = L::E, NPK = L::NPK, NTH = L::NTH,
                EQ = L::EQ, EV = L::EV, EF = L::EF, ETR = L::ETR, GEO = L::GEO,
                GF = L::GF;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S* sm = reinterpret_cast<S*>(smem_raw);
  int* sk = reinterpret_cast<int*>(sm + L::TOTAL);
  int* snc = sk + EB;
  S* sq = sm + L::SQ;
  S* sres = sm + L::SRES;
  S* sv = sm + L::SV;
  S* sfp = sm + L::SFP;
  S* sfu = sm + L::SFU;
  S* str = sm + L::STR;
  S* sg = sm + L::SG;
  S* smat = sm + L::SMAT;

  const hw_type_t& TY = M.t[T];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t w0 = (int64_t)blockIdx.x * EB;
  const int ne = (int)((nwork - w0) < EB ? (nwork - w0) : EB);
  const bool lsrk = E.mode == MODE_LSRK;
  // flux form from the type's form; the wedge volume is always the LSC-DG
  // skew two-pass (hybridwave/dg.py:423-444 has no strong branch)
  const bool skew = TY.form == HW_FORM_SKEW;
  const bool vskew = skew || T == HW_WEDGE;

  if (tid < EB) sk[tid] = tid < ne ? (list ? list[w0 + tid] : (int)(w0 + tid)) : 0;
  // zero K paddings (node rows NP..NPK and the per-face lift padding)
  constexpr int PADN = (NPK > NP) ? NPK - NP : 1;
  if (NPK > NP)
    for (int i = tid; i < EB * 11 * PADN; i += NTH) {
      const int e = i / (11 * PADN), r = i - e * 11 * PADN;
      const int fld = r / PADN, n = NP + r - fld * PADN;
      if (fld < 4) sq[e * EQ + fld * L::QF + n] = S(0);
      else if (fld >= 8) sv[e * EV + (fld - 8) * NPK + n] = S(0);
    }
  __syncthreads();

  // ---- P0: rows, records, links (all async), then neighbour staging
  const S* q = (const S*)Q.p[T];
  const S* resg = (const S*)E.res[T];
  copy_q_rows<L>(sq, q, sk, ne);
  {   // own traces of the input state (published by the previous stage)
    copy_rows16_w<4 * NFP, ETR, L::W>(str, (const S*)M.tr_in[T], sk, ne);
  }
  copy_rows_w<GEO, L::GEOS, L::W>(sg, (const S*)TY.geo, sk, ne);
  copy_rows<4, 4, NTH, EB>(smat, (const S*)TY.mat, sk, ne);
  for (int i = tid; i < ne * NF; i += NTH)
    snc[i] = __ldg(TY.nbr_code + (size_t)sk[i / NF] * NF + i % NF);
  cp_async_commit();
  // thread-item u = face point (e, j) = (tid + u * NTH) / NFP, % NFP (the
  // flux loop uses the same mapping)
  constexpr int IT = (EB * NFP + NTH - 1) / NTH;
  int gv[IT];
  R nb[IT][4];
  {
    // neighbour values at my face points through the host gather index
    // (already in my point order): index loads batched, then the values
    const bool sem = M.formulation == HW_SEM;
#pragma unroll
    for (int u = 0; u < IT; ++u) {
      const int i = tid + u * NTH;
      gv[u] = -1;
      if (i < ne * NFP) gv[u] = __ldg(TY.iop[1] + (size_t)sk[i / NFP] * NFP + i % NFP);
    }
    __syncthreads();                                // snc
#pragma unroll
    for (int u = 0; u < IT; ++u) {
      const int i = tid + u * NTH;
      if (i >= ne * NFP || gv[u] < 0) continue;
      const int e = i / NFP, j = i - e * NFP;
      int jj;
      const int f = face_of_point<N, T>(j, jj);
      const int t2 = HW_NBR_TYPE(snc[e * NF + f]);
      const S* src;
      int stride;
      if (publishes(t2, sem)) {
        src = (const S*)M.tr_in[t2];
        stride = nfp_of<N>(t2);
      } else if (t2 == HW_TET) {
        src = (const S*)Q.p[HW_TET];
        stride = Dims<N>::NP_TET;
      } else {
        src = (const S*)Q.p[HW_HEX];
        stride = Dims<N>::NP_HEX;
      }
      src += gv[u];
#pragma unroll
      for (int c = 0; c < 4; ++c) nb[u][c] = R(ldg(src + c * stride));
    }
    cp_async_commit();
  }
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");   // rows, records, own traces
  __syncthreads();

  // v_c = sum_x G[c][x] u_x
  for (int i = tid; i < ne * NP; i += NTH) {
    const int e = i / NP, n = i - e * NP;
    const S* G = sg + e * L::GEOS;
    const S* u = sq + e * EQ + n;
    const R u0 = u[L::QF], u1 = u[2 * L::QF], u2 = u[3 * L::QF];
#pragma unroll
    for (int c = 0; c < 3; ++c)
      sv[e * EV + c * NPK + n] = S(R(G[c * 3]) * u0 + R(G[c * 3 + 1]) * u1 + R(G[c * 3 + 2]) * u2);
  }
  __syncthreads();

  // ---- volume GEMMs
  const int grp = L::SPLIT ? warp / L::RT : 0, rt = warp - grp * L::RT;   // warp-uniform

  const int bk = lane & 3, bcol = lane >> 2;
  R dp[3][2] = {{0, 0}, {0, 0}, {0, 0}}, dv[2] = {0, 0};
  {
    const R* A = (const R*)TY.op[2];    // [3][RT][NPK/4][32] A_c fragments
    const R* AT = (const R*)TY.op[3];   // A_c^T fragments
    auto vol_u = [&]() {
      const S* bq = sq + bcol * EQ + bk;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const R* ac = A + (((c * L::RT + rt) * L::KPP) << 6) + 2 * lane;
        double2 pr;
#pragma unroll
        for (int ks = 0; ks < L::KSP; ++ks) {
          if (!(ks & 1)) pr = ldg2(ac + ((ks >> 1) << 6));
          dmma884(dp[c][0], dp[c][1], (ks & 1) ? pr.y : pr.x, bq[ks * 4]);
        }
      }
    };
    auto vol_p = [&]() {
      const S* bv = sv + bcol * EV + bk;
      const R* AV = vskew ? AT : A;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const R* ac = AV + (((c * L::RT + rt) * L::KPP) << 6) + 2 * lane;
        double2 pr;
#pragma unroll
        for (int ks = 0; ks < L::KSP; ++ks) {
          if (!(ks & 1)) pr = ldg2(ac + ((ks >> 1) << 6));
          dmma884(dv[0], dv[1], (ks & 1) ? pr.y : pr.x, bv[c * NPK + ks * 4]);
        }
      }
    };
    // split: the two groups take disjoint branches (if/else keeps their
    // register sets disjoint); otherwise one warp does both
    if (L::SPLIT) {
      if (grp == 0) vol_u(); else vol_p();
    } else {
      vol_u();
      vol_p();
    }
  }

  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();

  // ---- flux at the face points (face point fastest across threads)
  for (int i = tid; i < EB * L::NFKT; i += NTH) {   // lift K padding (storage held v_c)
    const int e = i / L::NFKT, k = i - e * L::NFKT;
    sfp[e * EF + k] = S(0);
    sfu[e * EF + k] = S(0);
  }
  __syncthreads();
  const R pen = R(M.penalty_scale);
#pragma unroll
  for (int u = 0; u < IT; ++u) {
    const int i = tid + u * NTH;
    if (i >= ne * NFP) break;
    const int e = i / NFP, j = i - e * NFP;
    int jj;
    const int f = face_of_point<N, T>(j, jj);
    const S* te = str + e * ETR + j;
    const R own[4] = {te[0], te[NFP], te[2 * NFP], te[3 * NFP]};
    const R um[3] = {own[1], own[2], own[3]};
    const S* g = sg + e * L::GEOS + GF + FS * f;
    const R nrm[3] = {g[0], g[1], g[2]};
    const int code = snc[e * NF + f];
    R pp, up[3];
    if (code & HW_NBR_BOUNDARY) {
      pp = -own[0]; up[0] = um[0]; up[1] = um[1]; up[2] = um[2];
    } else {
      pp = nb[u][0]; up[0] = nb[u][1]; up[1] = nb[u][2]; up[2] = nb[u][3];
    }
    R tp, tu, fp, fu;
    penalties(R(g[4]), R(g[5]), pen, tp, tu);
    upwind_flux(own[0], um, pp, up, nrm, tp, tu, skew, fp, fu);
    const int ko = L::koff_rt(f);
    sfp[e * EF + ko + jj] = S(fp * R(g[3]));
    sfu[e * EF + ko + jj] = S(fu * R(g[3]));
  }
  __syncthreads();
  // residual rows into the (now free) trace storage, behind the lift GEMM
  if (lsrk) {
    copy_q_rows<L>(sres, resg, sk, ne);
    cp_async_commit();
  }

  // ---- lift GEMMs, combine, epilogue (group 1: p rows, group 0: u rows)
  const int col0 = (lane & 3) * 2;
  const R* LF = (const R*)TY.op[4];     // [RT][NFKT/4][32] lift fragments
  R acc[3][2], accp[2];
  auto lift_p = [&]() {
    accp[0] = vskew ? dv[0] : -dv[0];
    accp[1] = vskew ? dv[1] : -dv[1];
    const S* bp = sfp + bcol * EF + bk;
    const R* lf = LF + ((rt * L::KPL) << 6) + 2 * lane;
    double2 pr;
#pragma unroll
    for (int j = 0; j < L::KSL; ++j) {
      if (!(j & 1)) pr = ldg2(lf + ((j >> 1) << 6));
      dmma884(accp[0], accp[1], (j & 1) ? pr.y : pr.x, bp[4 * j]);
    }
  };
  auto lift_u = [&]() {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const S* G = sg + (col0 + i) * L::GEOS;
#pragma unroll
      for (int x = 0; x < 3; ++x)
        acc[x][i] = -(R(G[x]) * dp[0][i] + R(G[3 + x]) * dp[1][i] + R(G[6 + x]) * dp[2][i]);
    }
    const S* bu = sfu + bcol * EF + bk;
    const R* lf = LF + ((rt * L::KPL) << 6) + 2 * lane;
    double2 pr;
    R tu[2] = {0, 0};
#pragma unroll
    for (int j = 0; j < L::KSL; ++j) {      // k-steps of all faces; fold per face
      if (!(j & 1)) pr = ldg2(lf + ((j >> 1) << 6));
      dmma884(tu[0], tu[1], (j & 1) ? pr.y : pr.x, bu[4 * j]);
      const int f = L::kface(j);
      if (j + 1 == L::KSL || L::kface(j + 1) != f) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const S* g = sg + (col0 + i) * L::GEOS + GF + FS * f;
          acc[0][i] += R(g[0]) * tu[i];
          acc[1][i] += R(g[1]) * tu[i];
          acc[2][i] += R(g[2]) * tu[i];
          tu[i] = R(0);
        }
      }
    }
  };
  if (L::SPLIT) {
    if (grp == 1) lift_p(); else lift_u();
  } else {
    lift_p();
    lift_u();
  }
  if (lsrk) {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
  }
  const int n = rt * 8 + (lane >> 2);
  if (n < NP) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int e = col0 + i;
      if (e >= ne) continue;
      const size_t base = (size_t)sk[e] * 4 * NP + n;
      S* qe = sq + e * EQ + n;
      const S* re = sres + e * EQ + n;
      auto out_p = [&]() {
        qe[0] = epilogue_q<S>(E, T, base,
                              S(accp[i] * R(smat[e * 4 + 0])) + frc_at<S>(E, T, base), qe[0],
                              re[0]);
      };
      auto out_u = [&]() {
        const R irho = R(smat[e * 4 + 1]);
#pragma unroll
        for (int x = 0; x < 3; ++x)
          qe[(1 + x) * L::QF] = epilogue_q<S>(E, T, base + (1 + x) * NP,
                                              S(acc[x][i] * irho) +
                                                  frc_at<S>(E, T, base + (1 + x) * NP),
                                              qe[(1 + x) * L::QF], re[(1 + x) * L::QF]);
      };
      if (L::SPLIT) {
        if (grp == 1) out_p(); else out_u();
      } else {
        out_p();
        out_u();
      }
    }
  }

  // ---- publish the traces of the new state: TR = E q_out
  if (E.mode != MODE_RHS && M.tr_out[T] != nullptr) {
    __syncthreads();
    publish_mma<L, T, S>(TY, sq, sg, sk, ne, (S*)M.tr_out[T]);
  }
}

// split layouts (RT <= HW_DENSE_SPLIT_MAX_RT): register target from MINB
template <int N, int T, typename S>
__global__ void __launch_bounds__(DMma<N, T, S>::NTH, DMma<N, T, S>::MINB)
    dense_mma_kernel(hw_mesh_t M, hw_fields_t Q, Epi E, const int32_t* __restrict__ list,
                     int64_t nwork) {
  dense_mma_body<N, T, S>(M, Q, E, list, nwork);
}

// large-RT layouts: register target of <= 64 per thread (N=5 wedge 560 ->
// 494 us, pyramid 113 -> 103 us; no change at N=4)
template <int N, int T, typename S>
__global__ void __launch_bounds__(DMma<N, T, S>::NTH, DMma<N, T, S>::BIG_MINB)
    dense_mma_kernel_big(hw_mesh_t M, hw_fields_t Q, Epi E, const int32_t* __restrict__ list,
                         int64_t nwork) {
  dense_mma_body<N, T, S>(M, Q, E, list, nwork);
}

// Face traces of q (hw_traces) for wedges / pyramids on DMMA: the
// epilogue's trace GEMM on the input rows.
template <int N, int T, typename S>
__global__ void __launch_bounds__(DMma<N, T, S>::NTH)
    trace_mma_kernel(hw_mesh_t M, hw_fields_t Q, hw_fields_t TR, const int32_t* __restrict__ list,
                     int64_t nwork) {
  using L = DMma<N, T, S>;
  constexpr int NP = L::NP, NPK = L::NPK, EB = L::E;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S* sq = reinterpret_cast<S*>(smem_raw);
  S* sg = sq + EB * L::EQ;
  int* sk = reinterpret_cast<int*>(sg + EB * L::GEOS + 2);
  const hw_type_t& TY = M.t[T];
  const int tid = threadIdx.x;
  const int64_t w0 = (int64_t)blockIdx.x * EB;
  const int ne = (int)((nwork - w0) < EB ? (nwork - w0) : EB);
  if (tid < EB) sk[tid] = tid < ne ? (list ? list[w0 + tid] : (int)(w0 + tid)) : 0;
  constexpr int PADN = (NPK > NP) ? NPK - NP : 1;
  if (NPK > NP)
    for (int i = tid; i < EB * 4 * PADN; i += L::NTH) {
      const int e = i / (4 * PADN), r = i - e * 4 * PADN;
      sq[e * L::EQ + (r / PADN) * L::QF + NP + r % PADN] = S(0);
    }
  __syncthreads();
  copy_q_rows<L>(sq, (const S*)Q.p[T], sk, ne);
  if (T == HW_WEDGE) copy_rows<L::GEO, L::GEOS, L::NTH, EB>(sg, (const S*)TY.geo, sk, ne);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  publish_mma<L, T, S>(TY, sq, sg, sk, ne, (S*)TR.p[T]);
}

}  // namespace hw
