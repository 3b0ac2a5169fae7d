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
  uint32_t size, hf_slot;
  uint32_t part_start[kSectorMaxParts + 1];  // CTA r holds S[part_start[r], part_start[r + 1])
  int n_ops, n_parts, f_real;
  uint64_t split_mask;          // generators flipping any of these qubits need a cluster barrier
  int32_t seg_off[kSectorMaxParts + 1];
  const int64_t* seg_start;     // [n_seg + 1]
  const int64_t* seg_foff;      // < 0: shared |f| (seg_fre/fim), else per-pair f offset
  const double* seg_fre;
  const double* seg_fim;
  const int64_t* gen_off;       // [CL * n_ops + 1], per op and owner rank
  const uint32_t* gen_pairs;    // slot_i | slot_j << 15 | sign << 30
  const uint8_t* gen_flags;     // pattern pair index << 1 (read only for multi-pattern ops)
  const uint32_t* exp_pairs;    // slot_i | slot_j << 15 | sign << 30
  const double* exp_fre;
  const double* exp_fim;  // nullptr when every f is real
};

// Amplitude slots (SectorProgram::slot_bits): 15 - log2(CL) offset bits, the
// owning rank above them. Addresses are 32-bit shared::cluster addresses (the
// shared::cta window when CL == 1).
template <int CL>
struct SlotMap {
  static constexpr int kBits = CL == 1 ? 15 : (CL == 2 ? 14 : (CL == 4 ? 13 : 12));
  uint32_t base[CL];
  __device__ __forceinline__ uint32_t addr(uint32_t s) const {
    const uint32_t off = (s & ((1u << kBits) - 1u)) << 4;
    if (CL == 1) return base[0] + off;
    const uint32_t r = (s >> kBits) & (CL - 1);
    uint32_t b = base[0];
#pragma unroll
    for (int q = 1; q < CL; ++q) b = r == (uint32_t)q ? base[q] : b;
    return b + off;
  }
};

template <int CL>
__device__ __forceinline__ double2 sld(uint32_t a) {
  double2 v;
  if (CL == 1)
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  else
    asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}

template <int CL>
__device__ __forceinline__ void sst(uint32_t a, double2 v) {
  if (CL == 1)
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y));
  else
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y));
}

// sum over one shared-|f| segment's pairs of sign * conj(psi[j]) psi[i]
// (.x real part, .y imaginary part unless FR); lane takes pairs s0 + lane + 32 u
template <int CL, bool FR>
__device__ __forceinline__ double2 seg_signed_sum(const uint32_t* __restrict__ pairs, int s0, int s1, int lane,
                                                  const SlotMap<CL>& sm) {
  double sr = 0.0, si = 0.0;
  for (int t = s0 + lane; t < s1; t += 128) {
    uint32_t w[4];
    double sg4[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int tu = t + 32 * u;
      w[u] = __ldg(pairs + min(tu, s1 - 1));
      sg4[u] = tu < s1 ? ((w[u] >> 30) ? -1.0 : 1.0) : 0.0;
    }
    double2 a[4], bb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = sld<CL>(sm.addr(w[u] & 0x7FFFu));
      bb[u] = sld<CL>(sm.addr((w[u] >> 15) & 0x7FFFu));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      sr = fma(sg4[u], fma(bb[u].x, a[u].x, bb[u].y * a[u].y), sr);
      if (!FR) si = fma(sg4[u], fma(bb[u].x, a[u].y, -bb[u].y * a[u].x), si);
    }
  }
  return make_double2(sr, si);
}

// one generator's pairs assigned to this CTA: exp(theta A) as the 2x2 rotation
// a' = c a + g F_hi b, b' = c b + g F_lo a per pair (g = +-s by the pair's sign)
template <int CL, int NT, bool MULTI>
__device__ __forceinline__ void gen_pass(const SectorDev& sd, const PlanDev& pl, int op, int64_t t0, int64_t t1,
                                         uint32_t w, double2 csv, double2 flo, double2 fhi, const SlotMap<CL>& sm) {
  for (int64_t t = t0; t < t1; t += NT) {
    if (t != t0) w = __ldg(sd.gen_pairs + t);
    if (MULTI) {  // more than one active pattern pair (not UCCSD)
      const int po = pl.fused[pl.op_idx[op]].pair_off + (__ldg(sd.gen_flags + t) >> 1);
      flo = pl.pair_f[2 * po];
      fhi = pl.pair_f[2 * po + 1];
    }
    const double g = (w >> 30) & 1u ? -csv.y : csv.y;
    const uint32_t pa = sm.addr(w & 0x7FFFu), pb = sm.addr((w >> 15) & 0x7FFFu);
    const double2 a = sld<CL>(pa), bb = sld<CL>(pb);
    const double2 hb = cmul(fhi, bb), la = cmul(flo, a);
    sst<CL>(pa, make_double2(csv.x * a.x + g * hb.x, csv.x * a.y + g * hb.y));
    sst<CL>(pb, make_double2(csv.x * bb.x + g * la.x, csv.x * bb.y + g * la.y));
  }
}

template <int CL, int NT>
__global__ void __launch_bounds__(NT, 1) k_sector_eval(SectorDev sd, PlanDev pl, const double* __restrict__ theta,
                                                       int theta_stride, double* __restrict__ e_out,
                                                       double* __restrict__ im_out, int n_rows,
                                                       long long* __restrict__ phase_clk) {
  // dynamic smem: [Hmax] amplitudes | [n_ops] (cos, sin*scale) | [n_ops] (F_lo, F_hi) of pattern pair 0 | [n_ops] flags
  extern __shared__ __align__(16) double2 sm_c[];
  __shared__ double2 red[NT / 32];
  __shared__ double cl_part[CL];
  const long long clk0 = clock64();
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = CL == 1 ? 0 : (int)cluster.block_rank();
  const int row = blockIdx.x / CL;
  if (row >= n_rows) return;  // whole clusters exit together (grid = n_rows * CL)
  uint32_t Hmax = 0;
#pragma unroll
  for (int r = 0; r < CL; ++r) Hmax = max(Hmax, sd.part_start[r + 1] - sd.part_start[r]);
  double2* cs = sm_c + Hmax;
  double2* fz = cs + pl.n_ops;  // [2 * n_ops]
  uint8_t* opfl = reinterpret_cast<uint8_t*>(fz + 2 * pl.n_ops);  // [n_ops]: bit 0 crosses the split, bit 1 multi-pattern
  SlotMap<CL> sm;
  {
    const uint32_t local = (uint32_t)__cvta_generic_to_shared(sm_c);
#pragma unroll
    for (int r = 0; r < CL; ++r) {
      if (CL == 1) {
        sm.base[r] = local;
      } else {
        uint32_t a;
        asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(local), "r"(r));
        sm.base[r] = a;
      }
    }
  }
  for (uint32_t i = threadIdx.x; i < Hmax; i += NT) sm_c[i] = make_double2(0.0, 0.0);
  for (int op = threadIdx.x; op < pl.n_ops; op += NT) {
    const double phi = theta[(int64_t)row * theta_stride + pl.op_gen[op]] * pl.op_cfac[op];
    double sv, cv;
    sincos(phi, &sv, &cv);
    cs[op] = make_double2(cv, sv * pl.op_sscale[op]);
    const FusedDesc& d = pl.fused[pl.op_idx[op]];
    fz[2 * op] = pl.pair_f[2 * d.pair_off];
    fz[2 * op + 1] = pl.pair_f[2 * d.pair_off + 1];
    opfl[op] = (uint8_t)(((d.x & sd.split_mask) != 0 ? 1 : 0) | (d.npair > 1 ? 2 : 0));
  }
  cluster.sync();
  if (threadIdx.x == 0 && (CL == 1 || (int)(sd.hf_slot >> SlotMap<CL>::kBits) == rank))
    sst<CL>(sm.addr(sd.hf_slot), make_double2(1.0, 0.0));
  cluster.sync();
  // generators: each CTA processes the pairs assigned to it (mostly local: S is
  // split on the qubits the fewest flip masks touch); one pair per thread per
  // trip, the next op's first pair word prefetched across the barrier
  const int tid = threadIdx.x;
  int64_t nx0 = sd.gen_off[rank] + tid, nx1 = sd.gen_off[rank + 1];  // op 0
  uint32_t nw = nx0 < nx1 ? __ldg(sd.gen_pairs + nx0) : 0u;
  for (int op = 0; op < sd.n_ops; ++op) {
    const int64_t t0 = nx0, t1 = nx1;
    uint32_t w = nw;
    if (op + 1 < sd.n_ops) {
      nx0 = sd.gen_off[CL * (op + 1) + rank] + tid;
      nx1 = sd.gen_off[CL * (op + 1) + rank + 1];
      nw = nx0 < nx1 ? __ldg(sd.gen_pairs + nx0) : 0u;
    }
    const int fl = opfl[op];
    if (t0 < t1) {
      if (fl & 2)
        gen_pass<CL, NT, true>(sd, pl, op, t0, t1, w, cs[op], fz[2 * op], fz[2 * op + 1], sm);
      else
        gen_pass<CL, NT, false>(sd, pl, op, t0, t1, w, cs[op], fz[2 * op], fz[2 * op + 1], sm);
    }
    // a generator whose flip mask avoids the split qubits only touches this
    // CTA's part: a CTA barrier suffices unless it or the next one crosses
    const bool cross = (fl & 1) != 0;
    const bool next_cross = op + 1 < sd.n_ops && (opfl[op + 1] & 1) != 0;
    if (CL > 1 && (cross || next_cross)) cluster.sync(); else __syncthreads();
  }
  const long long clk1 = clock64();
  // <H>: sum over (m, m ^ X) pairs of Re(conj(psi[j]) psi[i] f). Warp w takes
  // this rank's segments w, w + NT/32, ... (<= 512 pairs each); lanes take four
  // pairs per trip, every pair word and amplitude load issued before the
  // arithmetic; tail lanes re-read the last pair with weight 0 (no branches)
  double acc = 0.0;
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int sg = sd.seg_off[rank] + warp; sg < sd.seg_off[rank + 1]; sg += NT / 32) {
      const int s0 = (int)sd.seg_start[sg], s1 = (int)sd.seg_start[sg + 1];
      const int64_t foff = sd.seg_foff[sg];
      if (foff < 0) {  // shared |f|: per-pair sign, F applied once per segment
        if (sd.f_real)
          acc = fma(seg_signed_sum<CL, true>(sd.exp_pairs, s0, s1, lane, sm).x, sd.seg_fre[sg], acc);
        else {
          const double2 ss = seg_signed_sum<CL, false>(sd.exp_pairs, s0, s1, lane, sm);
          acc = fma(ss.x, sd.seg_fre[sg], fma(-ss.y, sd.seg_fim[sg], acc));
        }
      } else {  // per-pair f
        for (int t = s0 + lane; t < s1; t += 128) {
          uint32_t w[4];
          double fr[4], fi[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int tu = t + 32 * u;
            const int tc = min(tu, s1 - 1);
            w[u] = __ldg(sd.exp_pairs + tc);
            fr[u] = tu < s1 ? __ldg(sd.exp_fre + foff + (tc - s0)) : 0.0;
            fi[u] = (tu < s1 && sd.exp_fim) ? __ldg(sd.exp_fim + foff + (tc - s0)) : 0.0;
          }
          double2 a[4], bb[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            a[u] = sld<CL>(sm.addr(w[u] & 0x7FFFu));
            bb[u] = sld<CL>(sm.addr((w[u] >> 15) & 0x7FFFu));
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double prx = fma(bb[u].x, a[u].x, bb[u].y * a[u].y);
            const double pry = fma(bb[u].x, a[u].y, -bb[u].y * a[u].x);
            acc = fma(prx, fr[u], acc);
            acc = fma(-pry, fi[u], acc);
          }
        }
      }
    }
  }
  const double2 tot = block_sum<NT>(make_double2(acc, 0.0), red);
  // fixed-order cluster reduction: every rank writes its partial into rank 0
  if (CL == 1) {
    if (threadIdx.x == 0) cl_part[0] = tot.x;
  } else if (threadIdx.x == 0) {
    *cluster.map_shared_rank(&cl_part[rank], 0) = tot.x;
  }
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
