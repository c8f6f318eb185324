// Tet RHS + update with the dense contractions on the fp64 tensor cores
// (mma.sync.m8n8k4.f64, SASS DMMA), fp64 only.
//
// A block owns E tets; warp w owns one 8x8 output tile (row tile = 8 nodes,
// column tile = 8 elements).  All per-element smem arrays are element-major
// with an element stride = 4 (mod 16) doubles, so a B-fragment load (4
// consecutive k x 8 elements) touches every bank exactly twice (the minimum
// for 256 B) while whole element rows can be copied with 16-byte cp.async.
//   volume  DP_c = D_c p,  DIV = sum_c D_c v_c          (strong form)
//   lift    P += LIFT_f fp_f,  TU_f = LIFT_f fu_f,  U_x += n_f,x TU_f
// Neighbour face values come through a host-precomputed gather index in
// this element's face-point order (tet_gather_index in device.py), so the
// staging is one flat cp.async loop with no on-device orientation logic.
// On B200 DMMA and DFMA have the same peak (37 vs 34 TF/s measured); DMMA
// wins by needing 2 operand loads per 256 FMAs instead of ~1 per FMA.
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


template <int N>
struct TetMma {
  using D = Dims<N>;
  static constexpr int NP = D::NP_TET, NFN = D::NFN, NFP = 4 * D::NFN;
#ifndef HW_TET_E2
#define HW_TET_E2 16
#endif
#ifndef HW_TET_E4
#define HW_TET_E4 8
#endif
  static constexpr int E = (N == 1) ? 32 : (N == 2 ? HW_TET_E2 : (N == 4 ? HW_TET_E4 : 8));
  static constexpr int CT = E / 8;
  static constexpr int RT = (NP + 7) / 8;
  static constexpr int RT8 = RT * 8;
  static constexpr int NPK = ((NP + 3) / 4) * 4;
  static constexpr int NFK = ((NFN + 3) / 4) * 4;
  static constexpr int W = RT * CT;
  static constexpr int NTH = 32 * W;
  static constexpr bool VEC = (NP % 2 == 0) && (NPK == NP);  // 16-byte row copies
  static constexpr int EQ = stride4mod16(4 * NPK);          // q / res element stride
  static constexpr int EV = stride4mod16(3 * NPK);          // v_c
  static constexpr int EF = stride4mod16(4 * NFK);          // fp / fu
  static constexpr int ESG = 16 * NFN + 1;                  // staged neighbour values
  // buffers live in disjoint phases share storage: v_c (volume) with fp/fu
  // (flux, lift); the neighbour staging (flux) with the residual (epilogue)
#ifndef HW_TET_REGSTAGE
#define HW_TET_REGSTAGE 1
#endif
  // neighbour values: registers (REGSTAGE) or smem staging
  static constexpr int RA = cmax(EV, 2 * EF),
                       RB = stride4mod16(HW_TET_REGSTAGE ? EQ : cmax(16 * NFN, EQ));
  static constexpr int SQ = 0, SV = SQ + E * EQ, SFP = SV, SFU = SFP + E * EF,
                       SST = SV + E * RA, SRES = SST, SG = SST + E * RB,
                       SMAT = SG + E * GEO_TET, TOTAL = SMAT + E * 4;
  static constexpr size_t BYTES = sizeof(double) * TOTAL + sizeof(int) * (E + E * NFP + NFP);
#ifndef HW_TET_PERSIST
#define HW_TET_PERSIST 0
#endif
  // persistent blocks with register-resident operator fragments where they
  // fit (N <= 3: 27 doubles per thread)
  static constexpr bool PERSIST = HW_TET_PERSIST && (3 * (NPK / 4) + 4 * (NFK / 4)) <= 32;
#ifndef HW_TET_MINB
#define HW_TET_MINB 6
#endif
#ifndef HW_TET_PMINB
#define HW_TET_PMINB 4
#endif
  static constexpr int MINB = (W <= 4) ? (PERSIST ? HW_TET_PMINB : HW_TET_MINB) : ((W <= 8) ? 3 : 1);
};

template <int N>
__global__ void __launch_bounds__(TetMma<N>::NTH, TetMma<N>::MINB)
    tet_mma_kernel(hw_mesh_t M, hw_fields_t Q, Epi E, const int32_t* __restrict__ list,
                   int64_t nwork) {
  using L = TetMma<N>;
  using R = double;
  constexpr int NP = L::NP, NFN = L::NFN, NFP = L::NFP, EB = L::E, NPK = L::NPK,
                NFK = L::NFK, NTH = L::NTH, EQ = L::EQ, EV = L::EV, EF = L::EF,
                ESG = L::ESG;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sm = reinterpret_cast<R*>(smem_raw);
  int* sk = reinterpret_cast<int*>(sm + L::TOTAL);
  int* sgi = sk + EB;               // gather index [E][NFP]
  int* sfn = sgi + EB * NFP;        // own face node table
  R* sq = sm + L::SQ;
  R* sres = sm + L::SRES;
  R* sv = sm + L::SV;
  R* sfp = sm + L::SFP;
  R* sfu = sm + L::SFU;
  R* sst = sm + L::SST;
  R* sg = sm + L::SG;
  R* smat = sm + L::SMAT;

  const hw_type_t& TY = M.t[HW_TET];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool lsrk = E.mode == MODE_LSRK;
  for (int i = tid; i < NFP; i += NTH) sfn[i] = __ldg(TY.iop[0] + i);
  // persistent blocks: this warp's operator fragments (its row tile of D_c
  // and LIFT_f) stay in registers for every batch of elements it processes
  R Av[3][NPK / 4], Al[4][NFK / 4];
  if (L::PERSIST) {
    const int rt0 = warp / L::CT;
    const R* Dg = (const R*)TY.op[2];
    const R* Lg = (const R*)TY.op[3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int ks = 0; ks < NPK / 4; ++ks)
        Av[c][ks] = ldg(Dg + (((c * L::RT + rt0) * (NPK / 4) + ks) << 5) + lane);
#pragma unroll
    for (int f = 0; f < 4; ++f)
#pragma unroll
      for (int ks = 0; ks < NFK / 4; ++ks)
        Al[f][ks] = ldg(Lg + (((f * L::RT + rt0) * (NFK / 4) + ks) << 5) + lane);
  }
  const int64_t nbatch = (nwork + EB - 1) / EB;
  for (int64_t bidx = blockIdx.x; bidx < nbatch; bidx += (L::PERSIST ? gridDim.x : nbatch)) {
  const int64_t w0 = bidx * EB;
  const int ne = (int)((nwork - w0) < EB ? (nwork - w0) : EB);

  if (tid < EB) sk[tid] = tid < ne ? (list ? list[w0 + tid] : (int)(w0 + tid)) : 0;
  // K padding must be zero for the DMMA (rows are never written by copies)
  constexpr int PADN = (NPK > NP) ? NPK - NP : 1, PADF = (NFK > NFN) ? NFK - NFN : 1;
  if (NPK > NP)
    for (int i = tid; i < EB * 11 * PADN; i += NTH) {
      const int e = i / (11 * PADN), r = i - e * 11 * PADN;
      const int fld = r / PADN, n = NP + r - fld * PADN;
      if (fld < 4) sq[e * EQ + fld * NPK + n] = R(0);
      else if (fld >= 8) sv[e * EV + (fld - 8) * NPK + n] = R(0);
    }
  __syncthreads();

  // ---- P0: element rows (q, res), records and the gather index
  const R* q = (const R*)Q.p[HW_TET];
  const R* resg = (const R*)E.res[HW_TET];
  if (L::VEC) {
    copy_rows16<4 * NP, EQ, NTH, EB>(sq, q, sk, ne);
  } else {
    for (int i = tid; i < ne * 4 * NP; i += NTH) {
      const int e = i / (4 * NP), r = i - e * 4 * NP;
      const int fld = r / NP, n = r - fld * NP;
      cp_async(sq + e * EQ + fld * NPK + n, q + (size_t)sk[e] * 4 * NP + r);
    }
  }
  copy_rows<GEO_TET, GEO_TET, NTH, EB>(sg, (const R*)TY.geo, sk, ne);
  copy_rows<4, 4, NTH, EB>(smat, (const R*)TY.mat, sk, ne);
#if HW_TET_REGSTAGE
  // gather index straight into registers: thread-item u is (e, j) =
  // (tid + u * NTH) / NFP, % NFP, the same mapping the flux loop uses
  constexpr int IT = (EB * NFP + NTH - 1) / NTH;
  int gv[IT];
#pragma unroll
  for (int u = 0; u < IT; ++u) {
    const int i = tid + u * NTH;
    gv[u] = -1;
    if (i < ne * NFP) gv[u] = __ldg(TY.iop[1] + (size_t)sk[i / NFP] * NFP + i % NFP);
  }
#else
  if (NFP % 4 == 0)   // gather ints
    copy_rows16<NFP, NFP, NTH, EB>(sgi, TY.iop[1], sk, ne);
  else
    copy_rows<NFP, NFP, NTH, EB>(sgi, TY.iop[1], sk, ne);
#endif
  cp_async_commit();
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();

  // ---- P1: neighbour face-node values via the gather index
#if HW_TET_REGSTAGE
  R nb[IT][4];   // consumed by the flux after the volume GEMMs
#pragma unroll
  for (int u = 0; u < IT; ++u) {
    const int g = gv[u];
    if (g >= 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) nb[u][c] = ldg(q + (size_t)g + c * NP);
    } else if (g != -1) {   // pyramid / wedge neighbour: its published face trace
      const unsigned v = (unsigned)(-3 - g);
      const int t2 = (v & 1u) ? HW_WEDGE : HW_PYRAMID;
      const int nfp2 = (v & 1u) ? Dims<N>::NFP_WEDGE : Dims<N>::NFP_PYR;
      const R* src = (const R*)M.tr_in[t2] + (size_t)(v >> 1);
#pragma unroll
      for (int c = 0; c < 4; ++c) nb[u][c] = ldg(src + c * nfp2);
    }
  }
#else
  for (int i = tid; i < ne * NFP; i += NTH) {
    const int e = i / NFP, j = i - e * NFP;
    const int g = sgi[i];
    if (g == -1) continue;
    R* dst = sst + e * L::RB + j;            // [field][face point]: conflict-free
    if (g >= 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) cp_async(dst + c * NFP, q + (size_t)g + c * NP);
    } else {   // pyramid / wedge neighbour: its published face trace
      const unsigned v = (unsigned)(-3 - g);
      const int t2 = (v & 1u) ? HW_WEDGE : HW_PYRAMID;
      const int nfp2 = (v & 1u) ? Dims<N>::NFP_WEDGE : Dims<N>::NFP_PYR;
      const R* src = (const R*)M.tr_in[t2] + (size_t)(v >> 1);
#pragma unroll
      for (int c = 0; c < 4; ++c) cp_async(dst + c * NFP, src + c * nfp2);
    }
  }
  cp_async_commit();
#endif

  // v_c = sum_x G[c][x] u_x
  for (int i = tid; i < ne * NP; i += NTH) {
    const int e = i / NP, n = i - e * NP;
    const R* G = sg + e * GEO_TET;
    const R* u = sq + e * EQ + n;
    const R u0 = u[NPK], u1 = u[2 * NPK], u2 = u[3 * NPK];
#pragma unroll
    for (int c = 0; c < 3; ++c)
      sv[e * EV + c * NPK + n] = G[c * 3] * u0 + G[c * 3 + 1] * u1 + G[c * 3 + 2] * u2;
  }
  __syncthreads();

  // ---- P2: volume GEMMs on DMMA
  const int rt = warp / L::CT, ct = warp - rt * L::CT;

  const int bk = lane & 3, bcol = ct * 8 + (lane >> 2);
  R dp[3][2] = {{0, 0}, {0, 0}, {0, 0}}, dv[2] = {0, 0};
  {
    const R* Dg = (const R*)TY.op[2];   // [3][RT][NPK/4][32] A fragments, zero padded
    const R* bq = sq + bcol * EQ + bk;
    const R* bv = sv + bcol * EV + bk;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
      for (int ks = 0; ks < NPK / 4; ++ks) {
        const R a = L::PERSIST ? Av[c][ks]
                               : ldg(Dg + (((c * L::RT + rt) * (NPK / 4) + ks) << 5) + lane);
        dmma884(dp[c][0], dp[c][1], a, bq[ks * 4]);
        dmma884(dv[0], dv[1], a, bv[c * NPK + ks * 4]);
      }
    }
  }

  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();

  // ---- P3: flux at the face nodes (face point fastest across threads)
  if (NFK > NFN)      // K padding of fp/fu (their storage held v_c until now)
    for (int i = tid; i < EB * 8 * PADF; i += NTH) {
      const int e = i / (8 * PADF), r = i - e * 8 * PADF;
      const int fld = r / PADF, n = NFN + r - fld * PADF;
      (fld < 4 ? sfp : sfu)[e * EF + (fld & 3) * NFK + n] = R(0);
    }
  const R pen = R(M.penalty_scale);
#if HW_TET_REGSTAGE
#pragma unroll
  for (int u = 0; u < IT; ++u) {
    const int i = tid + u * NTH;
    if (i >= ne * NFP) break;
#else
  for (int i = tid; i < ne * NFP; i += NTH) {
#endif
    const int e = i / NFP, j = i - e * NFP;
    const int f = j / NFN, jj = j - f * NFN;
    const int node = sfn[j];
    const R* qe = sq + e * EQ + node;
    const R pm = qe[0];
    const R um[3] = {qe[NPK], qe[2 * NPK], qe[3 * NPK]};
    const R* g = sg + e * GEO_TET + 9 + FS * f;
    const R nrm[3] = {g[0], g[1], g[2]};
    R pp, up[3];
#if HW_TET_REGSTAGE
    if (gv[u] != -1) {
      pp = nb[u][0]; up[0] = nb[u][1]; up[1] = nb[u][2]; up[2] = nb[u][3];
    } else {
#else
    if (sgi[i] != -1) {
      const R* s = sst + e * L::RB + j;
      pp = s[0]; up[0] = s[NFP]; up[1] = s[2 * NFP]; up[2] = s[3 * NFP];
    } else {
#endif
      pp = -pm; up[0] = um[0]; up[1] = um[1]; up[2] = um[2];
    }
    R tp, tu, fp, fu;
    penalties(g[4], g[5], pen, tp, tu);
    upwind_flux(pm, um, pp, up, nrm, tp, tu, false, fp, fu);
    sfp[e * EF + f * NFK + jj] = fp * g[3];
    sfu[e * EF + f * NFK + jj] = fu * g[3];
  }
  __syncthreads();
  // residual rows into the (now free) staging storage, behind the lift GEMM
  if (lsrk) {
    if (L::VEC) {
      constexpr int CH = 4 * NP / 2;
      for (int i = tid; i < ne * CH; i += NTH) {
        const int e = i / CH, c = i - e * CH;
        cp_async16(sres + e * L::RB + 2 * c, resg + (size_t)sk[e] * 4 * NP + 2 * c);
      }
    } else {
      for (int i = tid; i < ne * 4 * NP; i += NTH) {
        const int e = i / (4 * NP), r = i - e * 4 * NP;
        const int fld = r / NP, n = r - fld * NP;
        cp_async(sres + e * L::RB + fld * NPK + n, resg + (size_t)sk[e] * 4 * NP + r);
      }
    }
    cp_async_commit();
  }

  // ---- P4: lift on DMMA, combine, epilogue
  const int col0 = ct * 8 + (lane & 3) * 2;
  R accp[2] = {-dv[0], -dv[1]};
  R accu[3][2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const R* G = sg + (col0 + i) * GEO_TET;
#pragma unroll
    for (int x = 0; x < 3; ++x)
      accu[x][i] = -(G[x] * dp[0][i] + G[3 + x] * dp[1][i] + G[6 + x] * dp[2][i]);
  }
  {
    const R* Lg = (const R*)TY.op[3];   // [4][RT][NFK/4][32] A fragments
    const R* bp = sfp + bcol * EF + bk;
    const R* bu = sfu + bcol * EF + bk;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      R tu[2] = {0, 0};
#pragma unroll
      for (int ks = 0; ks < NFK / 4; ++ks) {
        const R a = L::PERSIST ? Al[f][ks]
                               : ldg(Lg + (((f * L::RT + rt) * (NFK / 4) + ks) << 5) + lane);
        dmma884(accp[0], accp[1], a, bp[f * NFK + ks * 4]);
        dmma884(tu[0], tu[1], a, bu[f * NFK + ks * 4]);
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const R* g = sg + (col0 + i) * GEO_TET + 9 + FS * f;
        accu[0][i] += g[0] * tu[i];
        accu[1][i] += g[1] * tu[i];
        accu[2][i] += g[2] * tu[i];
      }
    }
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
      const R kap = smat[e * 4 + 0], irho = smat[e * 4 + 1];
      const size_t base = (size_t)sk[e] * 4 * NP + n;
      const R* qe = sq + e * EQ + n;
      const R* re = sres + e * L::RB + n;
      epilogue_s<R>(E, HW_TET, base, accp[i] * kap, qe[0], re[0]);
#pragma unroll
      for (int x = 0; x < 3; ++x)
        epilogue_s<R>(E, HW_TET, base + (1 + x) * NP, accu[x][i] * irho, qe[(1 + x) * NPK],
                      re[(1 + x) * NPK]);
    }
  }
  if (L::PERSIST) __syncthreads();   // the next batch reuses shared memory
  }
}

}  // namespace hw
