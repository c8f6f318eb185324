// Tet RHS + update with the dense contractions on the fp64 tensor cores
// (mma.sync.m8n8k4.f64, SASS DMMA), fp64 only.
//
// A block owns E tets; warp w owns one 8x8 output tile (row tile = 8 nodes,
// column tile = 8 elements) of every per-element field.  Data are staged in
// smem node-major ([field][node][element], element stride 1, node stride
// CS) so that the B-fragment loads of a warp hit every bank exactly twice.
//   volume  DP_c = D_c [p],  DIV = sum_c D_c [v_c]        (strong form)
//   lift    P += LIFT_f [fp_f],  TU_f = LIFT_f [fu_f],  U_x += n_f,x TU_f
// with the reference's arithmetic (hybridwave/dg.py:401-421, 326-354,
// 479-490) reorganised as in dense_kernel.  On B200 DMMA and DFMA have the
// same peak (37 vs 34 TF/s measured); DMMA wins by needing 2 operand loads
// per 256 FMAs instead of ~1 per FMA.
#pragma once
#include "hw_kernels.cuh"

namespace hw {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int N>
struct TetMma {
  using D = Dims<N>;
  static constexpr int NP = D::NP_TET, NFN = D::NFN, NFP = 4 * D::NFN;
  static constexpr int E = (N == 1) ? 32 : (N <= 4 ? 16 : 8);
  static constexpr int CT = E / 8;
  static constexpr int RT = (NP + 7) / 8;
  static constexpr int RT8 = RT * 8;
  static constexpr int NPK = ((NP + 3) / 4) * 4;
  static constexpr int NFK = ((NFN + 3) / 4) * 4;
  static constexpr int W = RT * CT;
  static constexpr int NTH = 32 * W;
  static constexpr int CS = (E == 8) ? 8 : E + 4;
  static constexpr int STG = 4 * 4 * NFN + 1;             // staged values per element (odd
                                                          // stride: conflict-free per element)
  // smem layout (doubles)
  static constexpr int SQ = 0;                            // [4][NPK][CS]
  static constexpr int SV = SQ + 4 * NPK * CS;            // [3][NPK][CS]
  static constexpr int SFP = SV + 3 * NPK * CS;           // [4][NFK][CS]
  static constexpr int SFU = SFP + 4 * NFK * CS;          // [4][NFK][CS]
  static constexpr int SRES = SFU + 4 * NFK * CS;         // [4][NPK][CS] (node-major)
  static constexpr int SG = SRES + 4 * NPK * CS;          // [E][GEO_TET]
  static constexpr int SMAT = SG + E * GEO_TET;           // [E][4]
  static constexpr int SST = SMAT + E * 4;                // [E][STG]
  static constexpr int TOTAL = SST + E * STG;
  // ints after the doubles: sk[E], codes[4E], neighbour index[4E], face
  // nodes[NFP], orientation permutations[6 NFN]
  static constexpr size_t BYTES =
      sizeof(double) * TOTAL + sizeof(int) * (E + 8 * E + NFP + 6 * NFN);
  static constexpr int MINB = (W <= 8) ? 3 : 1;
};

template <int N>
__global__ void __launch_bounds__(TetMma<N>::NTH, TetMma<N>::MINB)
    tet_mma_kernel(hw_mesh_t M, hw_fields_t Q, Epi E, const int32_t* __restrict__ list,
                   int64_t nwork) {
  using L = TetMma<N>;
  using R = double;
  constexpr int NP = L::NP, NFN = L::NFN, NFP = L::NFP, EB = L::E, CS = L::CS;
  constexpr int NPK = L::NPK, NFK = L::NFK, NTH = L::NTH;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sm = reinterpret_cast<R*>(smem_raw);
  int* sk = reinterpret_cast<int*>(sm + L::TOTAL);
  int* snc = sk + EB;
  int* sne = snc + 4 * EB;
  int* sfn = sne + 4 * EB;          // face node -> volume node
  int* sperm = sfn + NFP;           // triangle orientation permutations
  R* sq = sm + L::SQ;
  R* sv = sm + L::SV;
  R* sfp = sm + L::SFP;
  R* sfu = sm + L::SFU;
  R* sg = sm + L::SG;
  R* smat = sm + L::SMAT;

  const hw_type_t& TY = M.t[HW_TET];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t w0 = (int64_t)blockIdx.x * EB;
  const int ne = (int)((nwork - w0) < EB ? (nwork - w0) : EB);

  if (tid < EB) sk[tid] = tid < ne ? (list ? list[w0 + tid] : (int)(w0 + tid)) : -1;
  for (int i = tid; i < NFP; i += NTH) sfn[i] = __ldg(TY.iop[0] + i);
  for (int i = tid; i < 6 * NFN; i += NTH) sperm[i] = __ldg(M.perm_tri + i);
  // zero the padded K rows (node and face-point padding) once
  if (NPK > NP)
    for (int i = tid; i < 7 * (NPK - NP) * CS; i += NTH) {
      const int fld = i / ((NPK - NP) * CS), r = i - fld * (NPK - NP) * CS;
      sm[L::SQ + (fld * NPK + NP) * CS + r] = R(0);   // SQ and SV are adjacent
    }
  if (NFK > NFN)
    for (int i = tid; i < 8 * (NFK - NFN) * CS; i += NTH) {
      const int fld = i / ((NFK - NFN) * CS), r = i - fld * (NFK - NFN) * CS;
      sm[L::SFP + (fld * NFK + NFN) * CS + r] = R(0);  // SFP and SFU are adjacent
    }
  __syncthreads();

  // ---- P0: q (transposed to node-major) and res via cp.async; small
  // records with plain loads
  const R* q = (const R*)Q.p[HW_TET];
  for (int i = tid; i < ne * 4 * NP; i += NTH) {
    const int e = i / (4 * NP), r = i - e * 4 * NP;
    const int fld = r / NP, n = r - fld * NP;
    cp_async(sq + (fld * NPK + n) * CS + e, q + (size_t)sk[e] * 4 * NP + r);
  }
  if (E.mode == MODE_LSRK) {
    const R* res = (const R*)E.res[HW_TET];
    for (int i = tid; i < ne * 4 * NP; i += NTH) {
      const int e = i / (4 * NP), r = i - e * 4 * NP;
      const int fld = r / NP, n = r - fld * NP;
      cp_async(sm + L::SRES + (fld * NPK + n) * CS + e, res + (size_t)sk[e] * 4 * NP + r);
    }
  }
  cp_async_commit();
  for (int i = tid; i < ne * GEO_TET; i += NTH) {
    const int e = i / GEO_TET, r = i - e * GEO_TET;
    sg[i] = ldg((const R*)TY.geo + (size_t)sk[e] * GEO_TET + r);
  }
  for (int i = tid; i < ne * 4; i += NTH) {
    const int e = i >> 2, f = i & 3;
    smat[i] = ldg((const R*)TY.mat + (size_t)sk[e] * 4 + f);
    snc[i] = __ldg(TY.nbr_code + (size_t)sk[e] * 4 + f);
    sne[i] = __ldg(TY.nbr_elem + (size_t)sk[e] * 4 + f);
  }
  __syncthreads();

  // ---- P1: stage neighbour face-node values (tet neighbours; others take
  // the direct path in the flux loop)
  {
    using Dm = Dims<N>;
    for (int pr = warp; pr < ne * 4; pr += L::W) {
      const int e = pr >> 2, f = pr & 3;
      const int code = snc[pr];
      if ((code & HW_NBR_BOUNDARY) || HW_NBR_TYPE(code) != HW_TET) continue;
      const int k2 = sne[pr], f2 = HW_NBR_FACE(code);
      const R* q2 = (const R*)Q.p[HW_TET] + (size_t)k2 * 4 * NP;
      const int* fn = sfn + f2 * NFN;
      R* dst = sm + L::SST + e * L::STG + f * 4 * NFN;
      for (int i = lane; i < 4 * NFN; i += 32) {
        const int c = i / NFN, n = i - c * NFN;
        cp_async(dst + i, q2 + c * Dm::NP_TET + fn[n]);
      }
    }
    cp_async_commit();
  }
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");   // q, res landed
  __syncthreads();

  // v_c = sum_x G[c][x] u_x (node-major)
  for (int i = tid; i < NP * EB; i += NTH) {
    const int n = i / EB, e = i - n * EB;
    const R* G = sg + e * GEO_TET;
    const R u0 = sq[(1 * NPK + n) * CS + e], u1 = sq[(2 * NPK + n) * CS + e],
            u2 = sq[(3 * NPK + n) * CS + e];
#pragma unroll
    for (int c = 0; c < 3; ++c)
      sv[(c * NPK + n) * CS + e] = G[c * 3] * u0 + G[c * 3 + 1] * u1 + G[c * 3 + 2] * u2;
  }
  __syncthreads();

  // ---- P2: volume GEMMs on DMMA
  const int rt = warp / L::CT, ct = warp - rt * L::CT;
  const int arow = rt * 8 + (lane >> 2), acol = lane & 3;   // A fragment coords
  const int bk = lane & 3, bcol = ct * 8 + (lane >> 2);      // B fragment coords
  R dp[3][2] = {{0, 0}, {0, 0}, {0, 0}}, dv[2] = {0, 0};
  {
    const R* Dg = (const R*)TY.op[2];   // [3][RT8][NPK], zero padded
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
      for (int ks = 0; ks < NPK / 4; ++ks) {
        const R a = ldg(Dg + ((size_t)c * L::RT8 + arow) * NPK + ks * 4 + acol);
        const R bp = sq[(0 * NPK + ks * 4 + bk) * CS + bcol];
        const R bv = sv[(c * NPK + ks * 4 + bk) * CS + bcol];
        dmma884(dp[c][0], dp[c][1], a, bp);
        dmma884(dv[0], dv[1], a, bv);
      }
    }
  }

  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();

  // ---- P3: flux at the face nodes (element fastest across threads)
  const R pen = R(M.penalty_scale);
  for (int i = tid; i < NFP * EB; i += NTH) {
    const int j = i / EB, e = i - j * EB;
    if (e >= ne) continue;
    const int f = j / NFN, jj = j - f * NFN;
    const int node = sfn[j];
    const R pm = sq[(0 * NPK + node) * CS + e];
    const R um[3] = {sq[(1 * NPK + node) * CS + e], sq[(2 * NPK + node) * CS + e],
                     sq[(3 * NPK + node) * CS + e]};
    const R* g = sg + e * GEO_TET + 9 + FS * f;
    const R nrm[3] = {g[0], g[1], g[2]};
    const int code = snc[e * 4 + f];
    R pp, up[3];
    if (code & HW_NBR_BOUNDARY) {
      pp = -pm; up[0] = um[0]; up[1] = um[1]; up[2] = um[2];
    } else {
      if (HW_NBR_TYPE(code) == HW_TET) {
        const int p = sperm[HW_NBR_PERM(code) * NFN + jj];
        const R* s = sm + L::SST + e * L::STG + f * 4 * NFN;
        pp = s[p]; up[0] = s[NFN + p]; up[1] = s[2 * NFN + p]; up[2] = s[3 * NFN + p];
      } else {
        R tr[4];
        neighbour_trace<N, R>(M, Q, code, sne[e * 4 + f], jj, true, tr);
        pp = tr[0]; up[0] = tr[1]; up[1] = tr[2]; up[2] = tr[3];
      }
    }
    R tp, tu, fp, fu;
    penalties(g[4], pen, tp, tu);
    upwind_flux(pm, um, pp, up, nrm, tp, tu, TY.form == HW_FORM_SKEW, fp, fu);
    sfp[(f * NFK + jj) * CS + e] = fp * g[3];
    sfu[(f * NFK + jj) * CS + e] = fu * g[3];
  }
  __syncthreads();

  // ---- P4: lift on DMMA, combine, epilogue
  const int col0 = ct * 8 + (lane & 3) * 2;      // accumulator columns col0, col0+1
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
    const R* Lg = (const R*)TY.op[3];   // [4][RT8][NFK], zero padded
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      R tu[2] = {0, 0};
#pragma unroll
      for (int ks = 0; ks < NFK / 4; ++ks) {
        const R a = ldg(Lg + ((size_t)f * L::RT8 + arow) * NFK + ks * 4 + acol);
        const R bp = sfp[(f * NFK + ks * 4 + bk) * CS + bcol];
        const R bu = sfu[(f * NFK + ks * 4 + bk) * CS + bcol];
        dmma884(accp[0], accp[1], a, bp);
        dmma884(tu[0], tu[1], a, bu);
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
  const int n = rt * 8 + (lane >> 2);
  if (n < NP) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int e = col0 + i;
      if (e >= ne) continue;
      const R kap = smat[e * 4 + 0], irho = smat[e * 4 + 1];
      const size_t base = (size_t)sk[e] * 4 * NP + n;
      const R* re = sm + L::SRES + n * CS + e;
      epilogue_s<R>(E, HW_TET, base, accp[i] * kap, sq[(0 * NPK + n) * CS + e], re[0]);
#pragma unroll
      for (int x = 0; x < 3; ++x)
        epilogue_s<R>(E, HW_TET, base + (1 + x) * NP, accu[x][i] * irho,
                      sq[((1 + x) * NPK + n) * CS + e], re[(1 + x) * NPK * CS]);
    }
  }
}

}  // namespace hw
