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

struct SectorDev {
  uint32_t size, half, hf_idx;
  int n_ops;
  const int64_t* gen_off;
  const uint32_t* gen_pairs;
  const uint8_t* gen_flags;
  int64_t n_exp;
  const uint32_t* exp_pairs;
  const double* exp_fre;
  const double* exp_fim;  // nullptr when every f is real
};

template <int CL, int NT>
__global__ void __launch_bounds__(NT, 1) k_sector_eval(SectorDev sd, PlanDev pl, const double* __restrict__ theta,
                                                       int theta_stride, double* __restrict__ e_out,
                                                       double* __restrict__ im_out, int n_rows) {
  extern __shared__ __align__(16) double2 sm_c[];  // [half] amplitudes, then [n_ops] rotation coefficients
  __shared__ double2 red[NT / 32];
  __shared__ double cl_part[CL];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int row = blockIdx.x / CL;
  if (row >= n_rows) return;  // whole clusters exit together (grid = n_rows * CL)
  const uint32_t H = sd.half;
  double2* cs = sm_c + H;
  // base pointers of both halves (local smem and the peer CTA's, via DSMEM)
  double2* part[CL];
#pragma unroll
  for (int r = 0; r < CL; ++r) part[r] = cluster.map_shared_rank(sm_c, r);
  auto at = [&](uint32_t i) -> double2* {
    if (CL == 1) return sm_c + i;
    return i < H ? part[0] + i : part[1] + (i - H);
  };
  for (uint32_t i = threadIdx.x; i < H; i += NT) sm_c[i] = make_double2(0.0, 0.0);
  for (int op = threadIdx.x; op < pl.n_ops; op += NT) {
    const double phi = theta[(int64_t)row * theta_stride + pl.op_gen[op]] * pl.op_cfac[op];
    double sv, cv;
    sincos(phi, &sv, &cv);
    cs[op] = make_double2(cv, sv * pl.op_sscale[op]);
  }
  cluster.sync();
  if (rank == 0 && threadIdx.x == 0) *at(sd.hf_idx) = make_double2(1.0, 0.0);
  cluster.sync();
  const int tid = rank * NT + threadIdx.x;
  constexpr int NTC = CL * NT;
  for (int op = 0; op < sd.n_ops; ++op) {
    const double2 csv = cs[op];
    const double c = csv.x, sn = csv.y;
    const FusedDesc d = pl.fused[pl.op_idx[op]];
    const int64_t t0 = sd.gen_off[op], t1 = sd.gen_off[op + 1];
    for (int64_t t = t0 + tid; t < t1; t += NTC) {
      const uint32_t ij = sd.gen_pairs[t];
      const uint8_t fl = sd.gen_flags[t];
      const int p = fl >> 1;
      const double g = (fl & 1u) ? -sn : sn;
      const double2 flo = pl.pair_f[2 * (d.pair_off + p)], fhi = pl.pair_f[2 * (d.pair_off + p) + 1];
      double2* pa = at(ij & 0xFFFFu);
      double2* pb = at(ij >> 16);
      const double2 a = *pa, bb = *pb;
      const double2 hb = cmul(fhi, bb), la = cmul(flo, a);
      *pa = make_double2(c * a.x + g * hb.x, c * a.y + g * hb.y);
      *pb = make_double2(c * bb.x + g * la.x, c * bb.y + g * la.y);
    }
    cluster.sync();
  }
  // <H>: sum over (m, m ^ X) pairs of Re(conj(psi[j]) psi[i] f)
  double acc = 0.0;
  for (int64_t t = tid; t < sd.n_exp; t += NTC) {
    const uint32_t ij = sd.exp_pairs[t];
    const double2 a = *at(ij & 0xFFFFu), bb = *at(ij >> 16);
    const double prx = bb.x * a.x + bb.y * a.y;
    acc = fma(prx, sd.exp_fre[t], acc);
    if (sd.exp_fim) {
      const double pry = bb.x * a.y - bb.y * a.x;
      acc = fma(-pry, sd.exp_fim[t], acc);
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
  }
}

}  // namespace ffq
