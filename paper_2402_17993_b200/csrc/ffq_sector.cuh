// ffq_sector.cuh -- support-closure evaluator: one energy evaluation per
// thread-block cluster with the state's |S| amplitudes in distributed shared
// memory (see SectorProgram in ffq_compile.hpp).
//
// S (the amplitudes reachable from |hf> through the plan's pair maps) is
// theta-independent, and every amplitude outside it is identically zero, so
// the evaluation keeps exactly S on chip: 15 876 complex128 values = 254 KB
// at 18 qubits, split over the CL = 2 CTAs of a cluster. Generator g is one
// pass over its precompiled pairs (i, j) of S -- the (k, k ^ X) pairing of
// the dense pass restricted to S -- and consecutive generators are separated
// by a cluster barrier instead of a kernel launch. The expectation is one pass
// over the precompiled (m, m ^ X) pairs with their class sums f(m). Pair
// tables are shared by every evaluation of the batch (L2-resident); the only
// per-evaluation HBM traffic is theta in and E out.
#pragma once

#include <cooperative_groups.h>

#include "ffq_kernels.cuh"

namespace ffq {

namespace cg = cooperative_groups;

constexpr int kSectorMaxParts = 8;

struct SectorDev {
  uint32_t size, hf_idx;
  uint32_t part_start[kSectorMaxParts + 1];  // CTA r holds S[part_start[r], part_start[r + 1])
  int n_ops, n_parts;
  uint64_t split_mask;          // generators flipping any of these qubits need a cluster barrier
  int32_t seg_off[kSectorMaxParts + 1];
  const int64_t* seg_start;     // [n_seg + 1]
  const int64_t* seg_foff;      // < 0: shared |f| (seg_fre/fim), else per-pair f offset
  const double* seg_fre;
  const double* seg_fim;
  const int64_t* gen_off;       // [CL * n_ops + 1], per op and owner rank
  const uint32_t* gen_pairs;
  const uint8_t* gen_flags;
  const uint32_t* exp_pairs;
  const double* exp_fre;
  const double* exp_fim;  // nullptr when every f is real
};

template <int CL, int NT>
__global__ void __launch_bounds__(NT, 1) k_sector_eval(SectorDev sd, PlanDev pl, const double* __restrict__ theta,
                                                       int theta_stride, double* __restrict__ e_out,
                                                       double* __restrict__ im_out, int n_rows,
                                                       long long* __restrict__ phase_clk) {
  // dynamic smem: [half] amplitudes | [n_ops] (cos, sin*scale) | [n_ops] (F_lo, F_hi) of pattern pair 0
  extern __shared__ __align__(16) double2 sm_c[];
  __shared__ double2 red[NT / 32];
  __shared__ double cl_part[CL];
  const long long clk0 = clock64();
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int row = blockIdx.x / CL;
  if (row >= n_rows) return;  // whole clusters exit together (grid = n_rows * CL)
  uint32_t pstart[CL + 1];
  uint32_t Hmax = 0;
#pragma unroll
  for (int r = 0; r <= CL; ++r) pstart[r] = sd.part_start[r];
#pragma unroll
  for (int r = 0; r < CL; ++r) Hmax = max(Hmax, pstart[r + 1] - pstart[r]);
  double2* cs = sm_c + Hmax;
  double2* fz = cs + pl.n_ops;  // [2 * n_ops]
  uint8_t* crossf = reinterpret_cast<uint8_t*>(fz + 2 * pl.n_ops);  // [n_ops]
  // base pointers of the parts: this CTA's part through the plain shared
  // window (LDS/STS), the peers' through the distributed-shared window
  double2* part[CL];
#pragma unroll
  for (int r = 0; r < CL; ++r) part[r] = (r == rank) ? sm_c : cluster.map_shared_rank(sm_c, r);
  // unrolled select chain (no dynamic index into part[]: it stays in registers)
  auto at = [&](uint32_t i) -> double2* {
    if (CL == 1) return sm_c + i;
    double2* p = part[0];
    uint32_t base = 0;
#pragma unroll
    for (int q = 1; q < CL; ++q)
      if (i >= pstart[q]) { p = part[q]; base = pstart[q]; }
    return p + (i - base);
  };
  for (uint32_t i = threadIdx.x; i < Hmax; i += NT) sm_c[i] = make_double2(0.0, 0.0);
  for (int op = threadIdx.x; op < pl.n_ops; op += NT) {
    const double phi = theta[(int64_t)row * theta_stride + pl.op_gen[op]] * pl.op_cfac[op];
    double sv, cv;
    sincos(phi, &sv, &cv);
    cs[op] = make_double2(cv, sv * pl.op_sscale[op]);
    const FusedDesc& d = pl.fused[pl.op_idx[op]];
    fz[2 * op] = pl.pair_f[2 * d.pair_off];
    fz[2 * op + 1] = pl.pair_f[2 * d.pair_off + 1];
    crossf[op] = (uint8_t)((d.x & sd.split_mask) != 0);
  }
  cluster.sync();
  if (threadIdx.x == 0 && sd.hf_idx >= pstart[rank] && sd.hf_idx < pstart[rank + 1])
    *at(sd.hf_idx) = make_double2(1.0, 0.0);
  cluster.sync();
  // each CTA processes the pairs whose first member it owns (mostly local:
  // S is split on the qubit the fewest flip masks touch)
  const int tid = threadIdx.x;
  int64_t nx0 = sd.gen_off[rank] + tid, nx1 = sd.gen_off[rank + 1];  // op 0
  uint32_t nij = nx0 < nx1 ? sd.gen_pairs[nx0] : 0u;
  uint8_t nfl = nx0 < nx1 ? sd.gen_flags[nx0] : (uint8_t)0;
  for (int op = 0; op < sd.n_ops; ++op) {
    const double2 csv = cs[op];
    const double c = csv.x, sn = csv.y;
    const int64_t t0 = nx0, t1 = nx1;
    uint32_t ij = nij;
    uint8_t fl = nfl;
    if (op + 1 < sd.n_ops) {
      nx0 = sd.gen_off[CL * (op + 1) + rank] + tid;
      nx1 = sd.gen_off[CL * (op + 1) + rank + 1];
      nij = nx0 < nx1 ? __ldg(sd.gen_pairs + nx0) : 0u;
      nfl = nx0 < nx1 ? __ldg(sd.gen_flags + nx0) : (uint8_t)0;
    }
    for (int64_t t = t0; t < t1; t += NT) {
      if (t != t0) {
        ij = __ldg(sd.gen_pairs + t);
        fl = __ldg(sd.gen_flags + t);
      }
      double2 flo, fhi;
      if ((fl >> 1) == 0) {
        flo = fz[2 * op];
        fhi = fz[2 * op + 1];
      } else {  // more than one active pattern pair (not UCCSD)
        const int po = pl.fused[pl.op_idx[op]].pair_off + (fl >> 1);
        flo = pl.pair_f[2 * po];
        fhi = pl.pair_f[2 * po + 1];
      }
      const double g = (fl & 1u) ? -sn : sn;
      double2* pa = at(ij & 0xFFFFu);
      double2* pb = at(ij >> 16);
      const double2 a = *pa, bb = *pb;
      const double2 hb = cmul(fhi, bb), la = cmul(flo, a);
      *pa = make_double2(c * a.x + g * hb.x, c * a.y + g * hb.y);
      *pb = make_double2(c * bb.x + g * la.x, c * bb.y + g * la.y);
    }
    // a generator whose flip mask avoids the split qubits only touches this
    // CTA's part: a CTA barrier suffices unless it or the next one crosses
    const bool cross = crossf[op] != 0;
    const bool next_cross = op + 1 < sd.n_ops && crossf[op + 1] != 0;
    if (CL > 1 && (cross || next_cross)) cluster.sync(); else __syncthreads();
  }
  const long long clk1 = clock64();
  // <H>: sum over (m, m ^ X) pairs of Re(conj(psi[j]) psi[i] f); four pairs per
  // trip with every table and amplitude load issued before the arithmetic
  // warp w takes this rank's segment chunks w, w + NT/32, ... (<= 512 pairs each);
  // lanes stride the chunk four pairs at a time
  double acc = 0.0;
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int sg = sd.seg_off[rank] + warp; sg < sd.seg_off[rank + 1]; sg += NT / 32) {
      const int64_t s0 = sd.seg_start[sg], s1 = sd.seg_start[sg + 1];
      const int64_t foff = sd.seg_foff[sg];
      const double Fr = sd.seg_fre[sg], Fi = sd.seg_fim[sg];
      for (int64_t t = s0 + lane; t < s1; t += 128) {
        uint32_t ij[4];
        double fr[4], fi[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t tu = t + 32 * u;
          const bool ok = tu < s1;
          ij[u] = ok ? __ldg(sd.exp_pairs + tu) : 0u;
          if (foff < 0) {
            const double sg2 = (ij[u] >> 30) ? -1.0 : 1.0;
            fr[u] = ok ? sg2 * Fr : 0.0;
            fi[u] = ok ? sg2 * Fi : 0.0;
          } else {
            fr[u] = ok ? __ldg(sd.exp_fre + foff + (tu - s0)) : 0.0;
            fi[u] = (ok && sd.exp_fim) ? __ldg(sd.exp_fim + foff + (tu - s0)) : 0.0;
          }
        }
        double2 a[4], bb[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a[u] = *at(ij[u] & 0x7FFFu);
          bb[u] = *at((ij[u] >> 15) & 0x7FFFu);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double prx = bb[u].x * a[u].x + bb[u].y * a[u].y;
          const double pry = bb[u].x * a[u].y - bb[u].y * a[u].x;
          acc = fma(prx, fr[u], acc);
          acc = fma(-pry, fi[u], acc);
        }
      }
    }
  }
  const double2 tot = block_sum<NT>(make_double2(acc, 0.0), red);
  // fixed-order cluster reduction: every rank writes its partial into rank 0
  if (threadIdx.x == 0) *cluster.map_shared_rank(&cl_part[rank], 0) = tot.x;
  cluster.sync();
  if (rank == 0 && threadIdx.x == 0) {
    double e = 0.0;
#pragma unroll
    for (int r = 0; r < CL; ++r) e += cl_part[r];
    e_out[row] = e;
    if (im_out) im_out[row] = 0.0;
    if (phase_clk) {  // diagnostics (FFQ_PHASE_CLOCKS): generator / expectation cycles
      phase_clk[2 * row] = clk1 - clk0;
      phase_clk[2 * row + 1] = clock64() - clk1;
    }
  }
}

}  // namespace ffq

namespace ffq {

// ---- sparse row-wise matvec on a Krylov basis (lanczos_ground, energy_exact) ----
// y[r] = sum_e val[e] * (gen ? theta[gen[e]] : 1) * x[col[e]]; one warp per row,
// lanes stride the row, fixed shuffle tree (deterministic).
__global__ void k_csr_matvec(int64_t rows, const int64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                             const double* __restrict__ vre, const double* __restrict__ vim,
                             const int32_t* __restrict__ gen, const double* __restrict__ theta,
                             const double2* __restrict__ x, double2* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t e = rp[r] + lane; e < rp[r + 1]; e += 32) {
      double ar = vre[e], ai = vim[e];
      if (gen) {
        const double t = theta[gen[e]];
        ar *= t;
        ai *= t;
      }
      const double2 v = x[col[e]];
      acc.x = fma(ar, v.x, fma(-ai, v.y, acc.x));
      acc.y = fma(ar, v.y, fma(ai, v.x, acc.y));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc.x += __shfl_down_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_down_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) y[r] = acc;
  }
}

}  // namespace ffq
