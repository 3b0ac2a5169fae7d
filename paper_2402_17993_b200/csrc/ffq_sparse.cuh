// ffq_sparse.cuh -- support-tracked passes over the dense [batch][2^n] state.
//
// Each state row carries a support bitmap: bit k of word k>>5 is set whenever
// amplitude k may be non-zero (a conservative superset, so skipping unset
// pairs is exact for ANY state). UCCSD from |HF> only populates the
// (N_alpha, N_beta) sector -- 6% of the amplitudes at 18 qubits -- so the
// generator and expectation passes below read the bitmap (1/128 of the state
// bytes) and touch only pairs with a set bit. A dense state simply has every
// bit set and the passes degrade to the dense ones.
#pragma once

#include "ffq_kernels.cuh"

namespace ffq {

// bit o of the result = bit (o ^ L) of w  (L < 32)
__device__ __forceinline__ uint32_t xor_permute(uint32_t w, uint32_t L) {
  if (L & 1u) w = ((w & 0x55555555u) << 1) | ((w >> 1) & 0x55555555u);
  if (L & 2u) w = ((w & 0x33333333u) << 2) | ((w >> 2) & 0x33333333u);
  if (L & 4u) w = ((w & 0x0F0F0F0Fu) << 4) | ((w >> 4) & 0x0F0F0F0Fu);
  if (L & 8u) w = ((w & 0x00FF00FFu) << 8) | ((w >> 8) & 0x00FF00FFu);
  if (L & 16u) w = (w << 16) | (w >> 16);
  return w;
}

// support of |bits> for every row: all zero except one bit
__global__ void k_support_basis(uint32_t* __restrict__ sup, int64_t words, int batch, uint64_t bits) {
  const int64_t total = words * batch;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = t % words;
    sup[t] = (w == (int64_t)(bits >> 5)) ? (1u << (bits & 31u)) : 0u;
  }
}

// set the basis amplitude of every row of an all-zero slab (clean-slab path)
__global__ void k_set_basis_sparse(double2* __restrict__ psi, int n, int batch, uint64_t bits,
                                   int64_t rstride) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < batch; b += gridDim.x * blockDim.x)
    psi[(int64_t)b * rstride + (int64_t)bits] = make_double2(1.0, 0.0);
}

// zero every amplitude whose support bit is set: leaves the slab all-zero
// (a superset of the non-zeros is cleared) without a dense pass
__global__ void k_support_zero(double2* __restrict__ psi, const uint32_t* __restrict__ sup, int n,
                               int batch, int64_t rstride) {
  const int64_t words = (int64_t)batch << (n - 5);
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < words; w += warps) {
    const uint32_t bits = sup[w];
    const int64_t row = w >> (n - 5), wr = w & ((1LL << (n - 5)) - 1);
    if ((bits >> lane) & 1u) psi[row * rstride + ((wr << 5) | lane)] = make_double2(0.0, 0.0);
  }
}

// exact support of arbitrary data (after upload or a dense pass)
__global__ void k_support_from_state(const double2* __restrict__ psi, uint32_t* __restrict__ sup,
                                     int64_t total_amps) {
  const int lane = threadIdx.x & 31;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total_amps;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = psi[k];
    const uint32_t b = __ballot_sync(0xffffffffu, a.x != 0.0 || a.y != 0.0);
    if (lane == 0) sup[k >> 5] = b;
  }
}

// exp(theta A) of one fused generator on the support: one thread per support
// word of the low pattern member; candidates = pairs with either bit set.
__global__ void __launch_bounds__(256) k_fused_gen_support(
    double2* __restrict__ psi, uint32_t* __restrict__ sup, int n, FusedDesc d,
    const uint64_t* __restrict__ pair_bits, const uint32_t* __restrict__ pair_low,
    const double2* __restrict__ pair_f, const double2* __restrict__ cs, int cs_stride, int op,
    int64_t rstride) {
  const int b = blockIdx.y;
  double2* s = psi + (int64_t)b * rstride;
  uint32_t* bw = sup + ((int64_t)b << (n - 5));
  const double2 csv = cs[(int64_t)b * cs_stride + op];
  const double c = csv.x, sn = csv.y;
  const uint32_t L = (uint32_t)(d.x & 31u);
  const uint64_t XH = d.x >> 5;
  const int ub = n - 5 - d.whi;
  const int64_t per_pair = 1LL << ub;
  const int64_t total = per_pair * d.npair;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(t >> ub);
    const uint64_t v = (uint64_t)(t & (per_pair - 1));
    const uint64_t pb = pair_bits[d.pair_off + p];
    const uint64_t wi = insert_bits<uint64_t>(v, d.qpack_hi, d.whi) | (pb >> 5);
    const uint64_t wp = wi ^ XH;
    const uint32_t lm = pair_low[d.pair_off + p];
    const uint32_t sk = bw[wi];
    const uint32_t sp = (wp == wi) ? sk : bw[wp];
    uint32_t cand = (sk | xor_permute(sp, L)) & lm;
    if (!cand) continue;
    const double2 flo = pair_f[2 * (d.pair_off + p)], fhi = pair_f[2 * (d.pair_off + p) + 1];
    const uint32_t grown = cand;
    const uint64_t base = wi << 5;
    while (cand) {
      const uint32_t o = __ffs(cand) - 1;
      cand &= cand - 1;
      const uint64_t k = base | o, kb = k ^ d.x;
      const double2 a = s[k], bb = s[kb];
      const double g = sn * sgn_par(k & d.zout);
      const double2 hb = cmul(fhi, bb), la = cmul(flo, a);
      s[k] = make_double2(c * a.x + g * hb.x, c * a.y + g * hb.y);
      s[kb] = make_double2(c * bb.x + g * la.x, c * bb.y + g * la.y);
    }
    // both members of every touched pair may now be non-zero
    if (wp == wi) {
      const uint32_t add = (grown | xor_permute(grown, L)) & ~sk;
      if (add) atomicOr(&bw[wi], add);
    } else {
      const uint32_t addk = grown & ~sk, addp = xor_permute(grown, L) & ~sp;
      if (addk) atomicOr(&bw[wi], addk);
      if (addp) atomicOr(&bw[wp], addp);
    }
  }
}

// Re(conj(psi[m^X]) psi[m] b(m)) for one pair of group d, active pattern p
__device__ __forceinline__ double pair_term(const double2* __restrict__ s, uint32_t m,
                                            const GroupDesc& d, const HamDev& h, int p) {
  const double2 a = s[m], bb = s[m ^ (uint32_t)d.x];
  const double prx = bb.x * a.x + bb.y * a.y, pry = bb.x * a.y - bb.y * a.x;
  double fx = 0.0, fy = 0.0;
  for (int o = 0; o < d.ncls; ++o) {
    const double sg = sgn_par((uint64_t)(m & (uint32_t)h.cls_z[d.cls_off + o]));
    const double2 fo = h.cls_f[d.val_off + o * d.nact + p];
    fx = fma(sg, fo.x, fx);
    fy = fma(sg, fo.y, fy);
  }
  return prx * fx - pry * fy;
}

// the same with the amplitudes already gathered
__device__ __forceinline__ double pair_term_ab(double2 a, double2 bb, uint32_t m, const GroupDesc& d,
                                               const HamDev& h, int p) {
  const double prx = bb.x * a.x + bb.y * a.y, pry = bb.x * a.y - bb.y * a.x;
  double fx = 0.0, fy = 0.0;
  for (int o = 0; o < d.ncls; ++o) {
    const double sg = sgn_par((uint64_t)(m & (uint32_t)h.cls_z[d.cls_off + o]));
    const double2 fo = h.cls_f[d.val_off + o * d.nact + p];
    fx = fma(sg, fo.x, fx);
    fy = fma(sg, fo.y, fy);
  }
  return prx * fx - pry * fy;
}

// <psi|H|psi> on the support: item = (group, pattern, 2048-word range);
// candidates are m with pattern p whose own AND partner bits are set; a warp
// queue packs them so the class loop runs on full warps.
template <int NT>
__global__ void __launch_bounds__(NT) k_expect_support(const double2* __restrict__ psi,
                                                       const uint32_t* __restrict__ sup, int n,
                                                       HamDev h, const int32_t* __restrict__ it_g,
                                                       const int32_t* __restrict__ it_p,
                                                       const int64_t* __restrict__ it_w0,
                                                       const uint32_t* __restrict__ act_low,
                                                       double2* __restrict__ partial, int64_t rstride) {
  __shared__ uint32_t q_m[NT];
  __shared__ double2 red[NT / 32];
  const int64_t item = blockIdx.x;
  const int b = blockIdx.y;
  const double2* s = psi + (int64_t)b * rstride;
  const uint32_t* bw = sup + ((int64_t)b << (n - 5));
  const int g = it_g[item], p = it_p[item];
  const GroupDesc d = h.groups[g];
  const uint32_t L = (uint32_t)(d.x & 31u);
  const uint64_t XH = d.x >> 5;
  const uint64_t pb = h.act_bits[d.act_off + p];
  const uint32_t lm = act_low[d.act_off + p];
  const int64_t W = 1LL << (n - 5 - d.whi);
  const int64_t w0 = it_w0[item], w1 = min(W, w0 + h.sitem_words);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* wq = q_m + warp * 32;
  double acc = 0.0;
  // word indices: the fixed bits (flip bits >= 5 of the enumerated pattern)
  // are constant; the free bits advance by a masked increment, so a lane
  // steps to its next word in 3 integer ops (no per-word bit insertion)
  const uint32_t nwm = (uint32_t)((1ULL << (n - 5)) - 1ULL);
  uint32_t fixm = 0;
  for (int i = 0; i < d.whi; ++i) fixm |= 1u << ((d.qpack_hi >> (6 * i)) & 63u);
  const uint32_t freem = nwm & ~fixm, fixv = (uint32_t)(pb >> 5) & fixm;
  const uint32_t XHw = (uint32_t)XH;
  const int64_t span = w1 - w0;
  const int64_t warp_words = (span + NT / 32 - 1) / (NT / 32);
  const int64_t ws = w0 + warp * warp_words, we = min(w1, ws + warp_words);
  const uint32_t step = insert_bits<uint32_t>(32u, d.qpack_hi, d.whi);
  uint32_t wfree = insert_bits<uint32_t>((uint32_t)(ws + lane), d.qpack_hi, d.whi);
  if (d.ncls <= 2) {
    // few classes: each lane evaluates its own candidates (no queue round trips)
    for (int64_t v0 = ws; v0 < we; v0 += 32) {
      if (v0 + lane < we) {
        const uint32_t wi = wfree | fixv;
        uint32_t cand = bw[wi] & xor_permute(bw[wi ^ XHw], L) & lm;
        const uint32_t X32 = (uint32_t)d.x;
        while (cand) {
          // two candidates per trip: both gathers in flight before any arithmetic
          const uint32_t m0 = (wi << 5) | (uint32_t)(__ffs(cand) - 1);
          cand &= cand - 1;
          const bool two = cand != 0;
          const uint32_t m1 = two ? ((wi << 5) | (uint32_t)(__ffs(cand) - 1)) : m0;
          if (two) cand &= cand - 1;
          const double2 a0 = __ldcg(s + m0), b0 = __ldcg(s + (m0 ^ X32));
          const double2 a1 = __ldcg(s + m1), b1 = __ldcg(s + (m1 ^ X32));
          acc += pair_term_ab(a0, b0, m0, d, h, p);
          if (two) acc += pair_term_ab(a1, b1, m1, d, h, p);
        }
      }
      wfree = ((wfree | ~freem) + step) & freem;
    }
  } else {
    int qn = 0;
    for (int64_t v0 = ws; v0 < we; v0 += 32) {
      uint32_t cand = 0, wi = 0;
      if (v0 + lane < we) {
        wi = wfree | fixv;
        cand = bw[wi] & xor_permute(bw[wi ^ XHw], L) & lm;
      }
      wfree = ((wfree | ~freem) + step) & freem;
      while (__any_sync(0xffffffffu, cand != 0)) {
        const bool has = cand != 0;
        uint32_t e = 0;
        if (has) {
          e = (wi << 5) | (uint32_t)(__ffs(cand) - 1);
          cand &= cand - 1;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, has);
        const int rank = __popc(bal & ((1u << lane) - 1u));
        const int cnt = __popc(bal);
        const int room = 32 - qn;
        if (has && rank < room) wq[qn + rank] = e;
        __syncwarp();
        if (cnt >= room) {  // queue full: one pair per lane
          acc += pair_term(s, wq[lane], d, h, p);
          __syncwarp();
          if (has && rank >= room) wq[rank - room] = e;
          __syncwarp();
          qn = cnt - room;
        } else {
          qn += cnt;
        }
      }
    }
    if (lane < qn) acc += pair_term(s, wq[lane], d, h, p);
  }
  const double2 tot = block_sum<NT>(make_double2(acc, 0.0), red);
  if (threadIdx.x == 0) partial[(int64_t)b * gridDim.x + item] = tot;
}

}  // namespace ffq

namespace ffq {

// ---- persistent per-state evaluator (6 <= n <= 20) -----------------------------
// One CTA owns one state row for the whole energy evaluation: its support
// bitmap lives in shared memory, amplitudes stay in the dense HBM/L2 slab
// (which must be all-zero on entry and is left all-zero on exit), generators
// are separated by __syncthreads instead of kernel launches, and the grouped
// expectation runs on the same support. Candidate pairs are packed into
// 128-entry warp queues and drained 4 pairs per lane with every gather issued
// before any arithmetic, so each warp keeps 8 loads in flight.
constexpr int kPersistMaxQubits = 20;
constexpr int kQ = 128;  // queue entries per warp (4 per lane)

// 4 generator pairs per lane; entries (pattern << 27) | k, valid when i < cnt
__device__ __forceinline__ void gen_pairs4(double2* __restrict__ s, const uint64_t* wq, int lane, int cnt,
                                           const FusedDesc& d, const double2* __restrict__ pair_f,
                                           double c, double sn) {
  uint32_t k[4];
  double2 a[4], b[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int j = lane + 32 * i;
    k[i] = j < cnt ? (uint32_t)wq[j] : 0xFFFFFFFFu;
    if (k[i] != 0xFFFFFFFFu) {
      const uint32_t kk = k[i] & 0x07FFFFFFu;
      a[i] = __ldcg(s + kk);
      b[i] = __ldcg(s + (kk ^ (uint32_t)d.x));
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (k[i] == 0xFFFFFFFFu) continue;
    const uint32_t kk = k[i] & 0x07FFFFFFu, qp = k[i] >> 27;
    const double2 flo = pair_f[2 * (d.pair_off + qp)], fhi = pair_f[2 * (d.pair_off + qp) + 1];
    const double g = sn * sgn_par((uint64_t)(kk & (uint32_t)d.zout));
    const double2 hb = cmul(fhi, b[i]), la = cmul(flo, a[i]);
    __stcg(s + kk, make_double2(c * a[i].x + g * hb.x, c * a[i].y + g * hb.y));
    __stcg(s + (kk ^ (uint32_t)d.x), make_double2(c * b[i].x + g * la.x, c * b[i].y + g * la.y));
  }
}

// 4 expectation pairs per lane; entries (group << 40) | (pattern << 32) | m
__device__ __forceinline__ double exp_terms4(const double2* __restrict__ s, const uint64_t* wq, int lane,
                                             int cnt, const HamDev& h) {
  uint64_t e[4];
  double2 a[4], b[4];
  uint32_t x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int j = lane + 32 * i;
    e[i] = j < cnt ? wq[j] : ~0ULL;
    if (e[i] != ~0ULL) {
      const uint32_t m = (uint32_t)e[i];
      x[i] = (uint32_t)h.groups[(int)(e[i] >> 40)].x;
      a[i] = __ldcg(s + m);
      b[i] = __ldcg(s + (m ^ x[i]));
    }
  }
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (e[i] == ~0ULL) continue;
    const uint32_t m = (uint32_t)e[i];
    const int g = (int)(e[i] >> 40), p = (int)((e[i] >> 32) & 0xFFu);
    const int ncls = h.groups[g].ncls, cls_off = h.groups[g].cls_off, val_off = h.groups[g].val_off,
              nact = h.groups[g].nact;
    const double prx = b[i].x * a[i].x + b[i].y * a[i].y, pry = b[i].x * a[i].y - b[i].y * a[i].x;
    double fx = 0.0, fy = 0.0;
    for (int o = 0; o < ncls; ++o) {
      const double sg = sgn_par((uint64_t)(m & (uint32_t)h.cls_z[cls_off + o]));
      const double2 fo = h.cls_f[val_off + o * nact + p];
      fx = fma(sg, fo.x, fx);
      fy = fma(sg, fo.y, fy);
    }
    acc += prx * fx - pry * fy;
  }
  return acc;
}

// append this lane's candidate entry to the warp queue; returns true (and the
// caller drains kQ entries) when the queue filled up -- the lanes that did not
// fit are re-queued by queue_refill after the drain.
struct QPush {
  int rank, cnt, room;
};
__device__ __forceinline__ QPush queue_push(uint64_t* wq, int qn, bool has, uint64_t e, int lane) {
  const uint32_t bal = __ballot_sync(0xffffffffu, has);
  QPush r;
  r.rank = __popc(bal & ((1u << lane) - 1u));
  r.cnt = __popc(bal);
  r.room = kQ - qn;
  if (has && r.rank < r.room) wq[qn + r.rank] = e;
  __syncwarp();
  return r;
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_eval_persistent(int n, PlanDev pl, HamDev h, uint64_t hf_bits,
                                                           const uint32_t* __restrict__ pair_low,
                                                           const uint32_t* __restrict__ act_low,
                                                           const double* __restrict__ theta,
                                                           int theta_stride, double2* __restrict__ slab,
                                                           double* __restrict__ e_out,
                                                           double* __restrict__ im_out, int n_rows,
                                                           long long* __restrict__ phase_clk) {
  extern __shared__ __align__(16) uint32_t smem_u[];
  const long long clk0 = clock64();
  __shared__ double2 red[NT / 32];
  const int row = blockIdx.x;
  if (row >= n_rows) return;
  const int nwb = n - 5;
  const uint32_t nw = 1u << nwb;
  uint32_t* bm = smem_u;                                       // [nw] support words
  double2* cs = reinterpret_cast<double2*>(smem_u + nw);       // [n_ops]
  uint64_t* qall = reinterpret_cast<uint64_t*>(cs + pl.n_ops);  // [NT/32][kQ] warp queues
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t* wq = qall + warp * kQ;
  double2* s = slab + ((int64_t)blockIdx.x << n);

  for (uint32_t w = threadIdx.x; w < nw; w += NT)
    bm[w] = (w == (uint32_t)(hf_bits >> 5)) ? (1u << (hf_bits & 31u)) : 0u;
  for (int op = threadIdx.x; op < pl.n_ops; op += NT) {
    const double phi = theta[(int64_t)row * theta_stride + pl.op_gen[op]] * pl.op_cfac[op];
    double sv, cv;
    sincos(phi, &sv, &cv);
    cs[op] = make_double2(cv, sv * pl.op_sscale[op]);
  }
  if (threadIdx.x == 0) __stcg(s + hf_bits, make_double2(1.0, 0.0));
  __syncthreads();

  // ---- generators ----
  for (int op = 0; op < pl.n_ops; ++op) {
    const double2 csv = cs[op];
    if (pl.op_kind[op] == 0) {
      const FusedDesc d = pl.fused[pl.op_idx[op]];
      const uint32_t L = (uint32_t)(d.x & 31u), XH = (uint32_t)(d.x >> 5);
      const int ub = nwb - d.whi;
      const uint32_t total = (uint32_t)d.npair << ub;
      int qn = 0;
      for (uint32_t t0 = 0; t0 < total; t0 += NT) {
        const uint32_t t = t0 + threadIdx.x;
        uint32_t cand = 0, wi = 0, wp = 0;
        int p = 0;
        if (t < total) {
          p = (int)(t >> ub);
          const uint32_t v = t & ((1u << ub) - 1u);
          wi = insert_bits<uint32_t>(v, d.qpack_hi, d.whi) | (uint32_t)(pl.pair_bits[d.pair_off + p] >> 5);
          wp = wi ^ XH;
          cand = (bm[wi] | xor_permute(bm[wp], L)) & pair_low[d.pair_off + p];
        }
        const uint32_t grown = cand;
        while (__any_sync(0xffffffffu, cand != 0)) {
          const bool has = cand != 0;
          uint64_t e = 0;
          if (has) {
            e = ((uint64_t)p << 27) | (wi << 5) | (uint32_t)(__ffs(cand) - 1);
            cand &= cand - 1;
          }
          const QPush r = queue_push(wq, qn, has, e, lane);
          if (r.cnt >= r.room) {
            gen_pairs4(s, wq, lane, kQ, d, pl.pair_f, csv.x, csv.y);
            __syncwarp();
            if (has && r.rank >= r.room) wq[r.rank - r.room] = e;
            __syncwarp();
            qn = r.cnt - r.room;
          } else {
            qn += r.cnt;
          }
        }
        // both members of every touched pair may now be non-zero (pairs are
        // disjoint: no other thread of this step owns these bits)
        if (grown) {
          if (wp == wi) {
            atomicOr(&bm[wi], grown | xor_permute(grown, L));
          } else {
            atomicOr(&bm[wi], grown);
            atomicOr(&bm[wp], xor_permute(grown, L));
          }
        }
      }
      if (qn > 0) gen_pairs4(s, wq, lane, qn, d, pl.pair_f, csv.x, csv.y);
    } else {
      // general (non-fused) string: dense rotation by this CTA, then exact support
      const int si = pl.op_idx[op];
      const uint32_t x = (uint32_t)pl.str_x[si], z = (uint32_t)pl.str_z[si];
      const double2 w = ipow_d(pl.str_ny[si] + 1);
      const double c = csv.x, sn = csv.y;
      const uint32_t dim = 1u << n;
      if (x == 0) {
        for (uint32_t k = threadIdx.x; k < dim; k += NT) {
          const double2 a = __ldcg(s + k);
          const double sg = sn * sgn_par(k & z);
          __stcg(s + k, make_double2(c * a.x - sg * a.y, c * a.y + sg * a.x));
        }
      } else {
        const int hb = __ffs(x) - 1;
        for (uint32_t t = threadIdx.x; t < dim / 2; t += NT) {
          const uint32_t k = insert_zero<uint32_t>(t, hb), kp = k ^ x;
          const double2 a = __ldcg(s + k), bb = __ldcg(s + kp);
          const double sk2 = sn * sgn_par(k & z), sp2 = sn * sgn_par(kp & z);
          const double2 wb = cmul(w, bb), wa = cmul(w, a);
          __stcg(s + k, make_double2(c * a.x + sp2 * wb.x, c * a.y + sp2 * wb.y));
          __stcg(s + kp, make_double2(c * bb.x + sk2 * wa.x, c * bb.y + sk2 * wa.y));
        }
      }
      __syncthreads();
      for (uint32_t k0 = 0; k0 < dim; k0 += NT) {
        const uint32_t k = k0 + threadIdx.x;
        const double2 a = __ldcg(s + k);
        const uint32_t b = __ballot_sync(0xffffffffu, a.x != 0.0 || a.y != 0.0);
        if (lane == 0) bm[k >> 5] = b;
      }
    }
    __syncthreads();
  }

  const long long clk1 = clock64();
  // ---- expectation: pairs with both bits set ----
  // warp w owns (group, pattern) items w, w + NT/32, ...; lanes scan 32 support
  // words at a time and one queue spans items, so gathers and class loops run
  // on full warps and warps overlap their latencies.
  double acc = 0.0;
  {
    int qn = 0;
    for (int g = warp; g < h.n_groups; g += NT / 32) {
      const GroupDesc d = h.groups[g];
      const uint32_t L = (uint32_t)(d.x & 31u), XH = (uint32_t)(d.x >> 5);
      const uint32_t total = 1u << (nwb - d.whi);
      for (int p = 0; p < d.nact; ++p) {
        const uint32_t pbh = (uint32_t)(h.act_bits[d.act_off + p] >> 5);
        const uint32_t lm = act_low[d.act_off + p];
        const uint64_t tag = ((uint64_t)g << 40) | ((uint64_t)p << 32);
        for (uint32_t t0 = 0; t0 < total; t0 += 32) {
          const uint32_t t = t0 + lane;
          uint32_t cand = 0, wi = 0;
          if (t < total) {
            wi = insert_bits<uint32_t>(t, d.qpack_hi, d.whi) | pbh;
            cand = bm[wi] & xor_permute(bm[wi ^ XH], L) & lm;
          }
          while (__any_sync(0xffffffffu, cand != 0)) {
            const bool has = cand != 0;
            uint64_t e = 0;
            if (has) {
              e = tag | (wi << 5) | (uint32_t)(__ffs(cand) - 1);
              cand &= cand - 1;
            }
            const QPush r = queue_push(wq, qn, has, e, lane);
            if (r.cnt >= r.room) {
              acc += exp_terms4(s, wq, lane, kQ, h);
              __syncwarp();
              if (has && r.rank >= r.room) wq[r.rank - r.room] = e;
              __syncwarp();
              qn = r.cnt - r.room;
            } else {
              qn += r.cnt;
            }
          }
        }
      }
    }
    if (qn > 0) acc += exp_terms4(s, wq, lane, qn, h);
  }
  const double2 tot = block_sum<NT>(make_double2(acc, 0.0), red);
  if (threadIdx.x == 0) {
    e_out[row] = tot.x;
    if (im_out) im_out[row] = 0.0;
    if (phase_clk) {  // diagnostics (FFQ_PHASE_CLOCKS): generator / expectation cycles
      phase_clk[2 * row] = clk1 - clk0;
      phase_clk[2 * row + 1] = clock64() - clk1;
    }
  }
  // ---- leave the slab row all-zero for the next evaluation ----
  for (uint32_t w = threadIdx.x; w < nw; w += NT) {
    uint32_t bits = bm[w];
    while (bits) {
      const uint32_t o = __ffs(bits) - 1;
      bits &= bits - 1;
      __stcg(s + ((w << 5) | o), make_double2(0.0, 0.0));
    }
  }
}

}  // namespace ffq
