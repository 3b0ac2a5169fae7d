// Compact real sector layout for large UCCSD states (n > 26, BASELINE config 5).
//
// A spin-conserving UCCSD plan applied to |HF> keeps the state in the
// (N_alpha, N_beta) sector, and with real F on every generator the state is
// real (see k_sector_eval_real). Instead of the dense 2^n complex layout
// (64 GiB at 32 qubits, <= 4% of it ever non-zero), the state is held as a
// real [C(m, N_alpha)][C(m, N_beta)] matrix: row = rank of the alpha string
// (even qubits), column = rank of the beta string (odd qubits). That is
// 1.3 GB at 32 qubits, and a pass streams whole rows.
//
//  - A generator pass (one fused op: flip mask x, low pattern lo, outside-Z
//    mask zout) visits the low members k = (alpha, beta) with (alpha & x_a)
//    == lo_a and (beta & x_b) == lo_b; the partner is (alpha ^ x_a, beta ^ x_b)
//    and the JW sign factorises, (-1)^popc(k & zout) = row sign * column sign.
//    The 2x2 rotation is k_sector_eval_real's (same F, same fma order).
//  - A Hamiltonian term (x, z, c) adds Re(c i^ny) * S with
//    S = sum_k psi_k psi_{k^x} (-1)^popc((k^x) & z) over k with both members
//    in the sector (SPEC.md:419-427 expectation restricted to the sector; psi is
//    real, so a term with Re(c i^ny) = 0 contributes nothing). Terms sharing a
//    flip mask are one pass (the pair weight sums their signed w). Each pass's
//    CTA partials land in fixed slots; one fixed-order reduction gives the energy.
//
// Eligibility (compact_program): n even, m = n / 2 <= 16, every op a fused
// generator with one real pattern pair that keeps both spin counts.
// (Included by ffq_capi.cu inside its internal namespace.)

constexpr int kCompactThreads = 256;

struct CompactOp {  // one fused op over compressed alpha / beta strings
  uint32_t xa, la, za, xb, lb, zb;
};
struct CompactTerm {  // one Hamiltonian term of a flip-mask group
  uint32_t za, zb;
  double w;  // Re(c i^ny)
};
struct CompactGroup {  // terms sharing the flip mask (xa, xb): one pass
  uint32_t xa, xb;
  int32_t t0, nt;
};

// per-op rotation coefficients for one theta row: (cos phi, sin phi * F_hi, sin phi * F_lo)
__global__ void k_compact_coef(PlanDev pl, const double* __restrict__ theta, double* __restrict__ coef) {
  const int op = blockIdx.x * blockDim.x + threadIdx.x;
  if (op >= pl.n_ops) return;
  const double phi = theta[pl.op_gen[op]] * pl.op_cfac[op];
  double sv, cv;
  sincos(phi, &sv, &cv);
  const double sn = sv * pl.op_sscale[op];
  const FusedDesc& d = pl.fused[pl.op_idx[op]];
  coef[3 * op] = cv;
  coef[3 * op + 1] = sn * pl.pair_f[2 * d.pair_off + 1].x;
  coef[3 * op + 2] = sn * pl.pair_f[2 * d.pair_off].x;
}

__global__ void k_compact_set(double* __restrict__ psi, int64_t at) { psi[at] = 1.0; }

// One CTA per row (alpha string); columns four per thread per trip, every load
// of a trip issued before its stores (the pairs of one op are disjoint).
__global__ void __launch_bounds__(kCompactThreads) k_compact_gen(double* __restrict__ psi, int na, int nb,
                                                                 const uint32_t* __restrict__ stra,
                                                                 const uint32_t* __restrict__ strb,
                                                                 const uint16_t* __restrict__ ranka,
                                                                 const uint16_t* __restrict__ rankb, CompactOp o,
                                                                 const double* __restrict__ coef) {
  constexpr int T = kCompactThreads, U = 4;
  const int r = blockIdx.x;
  const uint32_t a = __ldg(stra + r);
  if ((a & o.xa) != o.la) return;
  const double c = coef[0], gh0 = coef[1], gl0 = coef[2];
  double* __restrict__ pi = psi + (int64_t)r * nb;
  double* __restrict__ pj = psi + (int64_t)__ldg(ranka + (a ^ o.xa)) * nb;
  const uint32_t sa = (uint32_t)__popc(a & o.za) & 1u;
  for (int c0 = threadIdx.x; c0 < nb; c0 += U * T) {
    int ci[U], cj[U];
    uint32_t sg[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int col = c0 + u * T;
      ok[u] = col < nb;
      ci[u] = cj[u] = col;
      sg[u] = sa;
      if (ok[u] && (o.xb | o.zb)) {
        const uint32_t b = __ldg(strb + col);
        ok[u] = (b & o.xb) == o.lb;
        sg[u] ^= (uint32_t)__popc(b & o.zb) & 1u;
        if (o.xb && ok[u]) cj[u] = __ldg(rankb + (b ^ o.xb));
      }
    }
    double x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x[u] = ok[u] ? pi[ci[u]] : 0.0;
      y[u] = ok[u] ? pj[cj[u]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ok[u]) {
        pi[ci[u]] = fma(sg[u] ? -gh0 : gh0, y[u], c * x[u]);
        pj[cj[u]] = fma(sg[u] ? -gl0 : gl0, x[u], c * y[u]);
      }
  }
}

// One flip-mask group: sum over its pairs of psi_k psi_{k^x} * sum_t w_t
// (-1)^popc((k^x) & z_t); the CTA partial goes to part[blockIdx.x]. MULTI =
// false: a one-term group (random strings), its term t1 passed by value.
template <bool MULTI>
__global__ void __launch_bounds__(kCompactThreads) k_compact_term(const double* __restrict__ psi, int na, int nb,
                                                                  const uint32_t* __restrict__ stra,
                                                                  const uint32_t* __restrict__ strb,
                                                                  const uint16_t* __restrict__ ranka,
                                                                  const uint16_t* __restrict__ rankb, CompactGroup gr,
                                                                  const CompactTerm* __restrict__ terms,
                                                                  CompactTerm t1, double2* __restrict__ part) {
  __shared__ double2 red[kCompactThreads / 32];
  const int ha = __popc(gr.xa) / 2, hb = __popc(gr.xb) / 2;
  const CompactTerm* tt = terms + gr.t0;
  double acc = 0.0;
  for (int r = blockIdx.x; r < na; r += gridDim.x) {
    const uint32_t a = __ldg(stra + r);
    if (__popc(a & gr.xa) != ha) continue;
    const uint32_t ap = a ^ gr.xa;
    const int64_t ri = (int64_t)r * nb, rj = (int64_t)__ldg(ranka + ap) * nb;
    double racc = 0.0;
    constexpr int U = 4;
    for (int c0 = threadIdx.x; c0 < nb; c0 += U * kCompactThreads) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int col = c0 + u * kCompactThreads;
        v[u] = 0.0;
        if (col < nb) {
          const uint32_t b = __ldg(strb + col);
          if (__popc(b & gr.xb) == hb) {
            const uint32_t bp = b ^ gr.xb;
            const int cj = gr.xb ? __ldg(rankb + bp) : col;
            const double p = psi[ri + col] * psi[rj + cj];
            if (!MULTI) {
              const uint32_t s = ((uint32_t)__popc(ap & t1.za) ^ (uint32_t)__popc(bp & t1.zb)) & 1u;
              v[u] = s ? -t1.w * p : t1.w * p;
            } else {
              double f = 0.0;
              for (int t = 0; t < gr.nt; ++t) {
                const uint32_t s = ((uint32_t)__popc(ap & tt[t].za) ^ (uint32_t)__popc(bp & tt[t].zb)) & 1u;
                f += s ? -tt[t].w : tt[t].w;
              }
              v[u] = f * p;
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) racc += v[u];
    }
    acc += racc;
  }
  const double2 tot = block_sum<kCompactThreads>(make_double2(acc, 0.0), red);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

struct CompactProg {
  bool ok = false;
  int m = 0, na = 0, nb = 0;
  int64_t hf_at = 0;
  std::vector<CompactOp> ops;
  std::vector<CompactGroup> groups;  // flip-mask groups of the terms that can contribute
  std::vector<CompactTerm> host_terms;
  DevBuf<CompactTerm> terms;
  DevBuf<uint32_t> stra, strb;
  DevBuf<uint16_t> ranka, rankb;
};

// bits of x selected by mask, packed low
inline uint32_t compact_pext(uint64_t x, uint64_t mask) {
  uint32_t out = 0;
  int k = 0;
  for (int q = 0; q < 64; ++q)
    if ((mask >> q) & 1u) out |= (uint32_t)((x >> q) & 1u) << k++;
  return out;
}

inline std::vector<uint32_t> strings_with(int m, int k) {
  std::vector<uint32_t> out;
  for (uint32_t s = 0; s < (1u << m); ++s)
    if (__builtin_popcount(s) == k) out.push_back(s);
  return out;
}

// nullptr when the plan / Hamiltonian / HF state does not fit the compact layout
CompactProg* compact_program(ffq_ctx_t ctx, ffq_plan_s* pl, ffq_ham_s* h, uint64_t hf) {
  const int n = pl->cp.n_qubits;
  const std::string key = "compact:" + std::to_string(h->uid) + ":" + std::to_string(hf);
  auto it = pl->compacts.find(key);
  if (it != pl->compacts.end()) {
    CompactProg* c = static_cast<CompactProg*>(it->second.get());
    return c->ok ? c : nullptr;
  }
  auto cp = std::make_shared<CompactProg>();
  const CompiledPlan& P = pl->cp;
  const uint64_t ev = 0x5555555555555555ull & ((n >= 64) ? ~0ull : ((1ull << n) - 1ull)), od = ev << 1;
  bool ok = n % 2 == 0 && n / 2 <= 16 && plan_is_real(P) && !P.op_kind.empty();
  for (size_t op = 0; ok && op < P.op_kind.size(); ++op) {
    const FusedDesc& d = P.fused[P.op_idx[op]];
    const uint64_t lo = P.pair_bits[d.pair_off];
    CompactOp o{compact_pext(d.x, ev), compact_pext(lo, ev), compact_pext(d.zout, ev),
                compact_pext(d.x, od), compact_pext(lo, od), compact_pext(d.zout, od)};
    ok = 2 * __builtin_popcount(o.la) == __builtin_popcount(o.xa) &&
         2 * __builtin_popcount(o.lb) == __builtin_popcount(o.xb);
    cp->ops.push_back(o);
  }
  if (ok) {
    const int m = n / 2, ka = __builtin_popcountll(hf & ev), kb = __builtin_popcountll(hf & od);
    const std::vector<uint32_t> sa = strings_with(m, ka), sb = strings_with(m, kb);
    std::vector<uint16_t> ra(1u << m, 0), rb(1u << m, 0);
    for (size_t i = 0; i < sa.size(); ++i) ra[sa[i]] = (uint16_t)i;
    for (size_t i = 0; i < sb.size(); ++i) rb[sb[i]] = (uint16_t)i;
    cp->m = m;
    cp->na = (int)sa.size();
    cp->nb = (int)sb.size();
    cp->hf_at = (int64_t)ra[compact_pext(hf, ev)] * cp->nb + rb[compact_pext(hf, od)];
    std::map<uint64_t, std::vector<CompactTerm>> by_x;  // (xa, xb) -> terms, in upload order
    for (size_t t = 0; t < h->raw_x.size(); ++t) {
      const uint64_t x = h->raw_x[t], z = h->raw_z[t];
      const int ny = __builtin_popcountll(x & z) & 3;
      // Re(c i^ny)
      const double w = ny == 0 ? h->raw_re[t] : ny == 1 ? -h->raw_im[t] : ny == 2 ? -h->raw_re[t] : h->raw_im[t];
      const uint32_t xa = compact_pext(x, ev), xb = compact_pext(x, od);
      if (w == 0.0 || __builtin_popcount(xa) % 2 || __builtin_popcount(xb) % 2) continue;
      if (__builtin_popcount(xa) / 2 > std::min(ka, m - ka) || __builtin_popcount(xb) / 2 > std::min(kb, m - kb))
        continue;  // no sector member can pair with a sector member
      by_x[((uint64_t)xa << 32) | xb].push_back({compact_pext(z, ev), compact_pext(z, od), w});
    }
    std::vector<CompactTerm>& tl = cp->host_terms;
    for (const auto& kv : by_x) {
      cp->groups.push_back({(uint32_t)(kv.first >> 32), (uint32_t)kv.first, (int32_t)tl.size(),
                            (int32_t)kv.second.size()});
      tl.insert(tl.end(), kv.second.begin(), kv.second.end());
    }
    cp->terms.upload(tl, ctx->stream);
    cp->stra.upload(sa, ctx->stream);
    cp->strb.upload(sb, ctx->stream);
    cp->ranka.upload(ra, ctx->stream);
    cp->rankb.upload(rb, ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
  }
  cp->ok = ok;
  auto* raw = cp.get();
  pl->compacts.emplace(key, std::move(cp));
  return ok ? raw : nullptr;
}

// energies of `batch` theta rows (device) into e/im (device), one state at a time
void compact_energy(ffq_ctx_t ctx, ffq_plan_s* pl, CompactProg& cp, const double* theta, int batch, double* e,
                    double* im) {
  const size_t dim = (size_t)cp.na * cp.nb;
  ctx->compact_psi.alloc(dim);
  ctx->compact_coef.alloc(3 * pl->cp.op_kind.size());
  const int g = 32 * ctx->n_sm;  // term kernels: fixed grid (fixed partial slots)
  const size_t nterm = cp.groups.size();
  ctx->compact_part.alloc(std::max<size_t>(1, nterm * g));
  const PlanDev pd = pl->dev();
  const int nops = (int)pl->cp.op_kind.size();
  for (int b = 0; b < batch; ++b) {
    CK(cudaMemsetAsync(ctx->compact_psi.p, 0, dim * sizeof(double), ctx->stream));
    k_compact_set<<<1, 1, 0, ctx->stream>>>(ctx->compact_psi.p, cp.hf_at);
    k_compact_coef<<<(nops + 127) / 128, 128, 0, ctx->stream>>>(pd, theta + (size_t)b * pl->cp.n_gen,
                                                               ctx->compact_coef.p);
    for (int op = 0; op < nops; ++op)
      k_compact_gen<<<cp.na, kCompactThreads, 0, ctx->stream>>>(ctx->compact_psi.p, cp.na, cp.nb, cp.stra.p, cp.strb.p,
                                                             cp.ranka.p, cp.rankb.p, cp.ops[op],
                                                             ctx->compact_coef.p + 3 * op);
    for (size_t t = 0; t < nterm; ++t)
      (cp.groups[t].nt == 1 ? k_compact_term<false> : k_compact_term<true>)<<<g, kCompactThreads, 0, ctx->stream>>>(
          ctx->compact_psi.p, cp.na, cp.nb, cp.stra.p, cp.strb.p, cp.ranka.p, cp.rankb.p, cp.groups[t], cp.terms.p,
          cp.host_terms[cp.groups[t].t0], ctx->compact_part.p + t * g);
    if (nterm == 0) CK(cudaMemsetAsync(ctx->compact_part.p, 0, sizeof(double2), ctx->stream));
    k_reduce_partials<kThreads><<<1, kThreads, 0, ctx->stream>>>(ctx->compact_part.p,
                                                                  (int64_t)std::max<size_t>(1, nterm * g), e + b,
                                                                  im ? im + b : nullptr);
    CK(cudaGetLastError());
    ctx->launches += 4 + nops + (int64_t)nterm;
  }
}
