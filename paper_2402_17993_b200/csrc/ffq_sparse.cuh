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
