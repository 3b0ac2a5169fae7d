// ffq_shard.inl -- sharded state vector (BASELINE.json config 5).
// Included at the end of ffq_capi.cu (same translation unit).
//
// A state of n qubits is split on its g highest *physical* qubits over
// R = 2^g ranks; rank r holds the 2^l amplitudes (l = n - g) whose physical
// index is (r << l) | k. Plan ops whose flip mask reaches a global position
// are preceded by a qubit swap with a free local position (schedule_shards):
// ranks r and r ^ (1 << j) exchange the half shard whose local bit differs
// from their rank bit. Z on global qubits is a per-rank sign folded into sin.
// Generator passes are support-tracked per shard (bitmaps rebuilt after a swap).
// The expectation exchanges whole shards once per distinct out-of-shard flip
// pattern hG and evaluates that bucket of x-groups locally.
//
// Transport: "group" mode keeps all R shards on one device (exchanges are
// device-side swaps; used for 1-GPU validation); "nccl" mode is one shard per
// process with ncclSend/ncclRecv over NVLink and an allgather of the per-rank
// partial energies summed in rank order (deterministic).
#include <nccl.h>

struct ffq_shard_s {
  ffq_ctx_t ctx = nullptr;
  int n = 0, g = 0, l = 0, R = 1;
  int rank = -1;  // nccl mode: this process's rank; group mode: -1
  std::vector<std::unique_ptr<DevBuf<double2>>> shards;  // group: R, nccl: 1
  DevBuf<double2> sendbuf, recvbuf;
  DevBuf<double2> cs, partial;
  DevBuf<double> eloc;
  DevBuf<uint64_t> pbits;
  DevBuf<uint32_t> plow;  // low_pattern_mask of every pattern pair at its op's physical positions
  ncclComm_t comm = nullptr;
  std::vector<int> perm;
  int last_swaps = 0;
  // cache: physical Hamiltonian per (ham, final perm)
  uint64_t ham_key = 0;  // ffq_ham_s::uid of the cached physical Hamiltonian
  std::vector<int> ham_perm;
  std::unique_ptr<ffq_ham_s> hphys;
  // one-term groups with |X| > 6 (random Pauli strings), batched per out-of-shard
  // flip pattern (k_expect_shard_multi): terms, batches of <= 16, buckets
  DevBuf<ShardTerm> mterms;
  DevBuf<int2> mbatches;
  DevBuf<uint32_t> sup_own, sup_partner;  // support bitmaps of the local shards / of a received partner shard
  DevBuf<uint32_t> sendidx, recvidx;      // support-compacted swaps: indices within the half
  DevBuf<unsigned long long> counters;    // [4]: counts and cursors of a swap
  int64_t sparse_swaps = 0, dense_swaps = 0;
  struct MultiBucket {
    uint32_t hG;
    int batch0, n_batches;
  };
  std::vector<MultiBucket> mbuckets;
  int64_t mchunk = 0, mchunks = 0;  // bitmap words per CTA, CTAs per batch
  ~ffq_shard_s() {
    if (comm) ncclCommDestroy(comm);
  }
  bool group() const { return rank < 0; }
  int n_local() const { return group() ? R : 1; }
  int rank_of(int i) const { return group() ? i : rank; }
};

namespace {

#define NCK(call)                                                                      \
  do {                                                                                 \
    ncclResult_t r_ = (call);                                                          \
    if (r_ != ncclSuccess)                                                             \
      throw NcclError(std::string(#call) + ": " + ncclGetErrorString(r_));             \
  } while (0)

struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <typename F>
int guarded_shard(ffq_ctx_t ctx, F&& f) {
  try {
    return guarded(ctx, f);
  } catch (const NcclError& e) {
    return fail(ctx, FFQ_ENCCL, e.what());
  }
}

void shard_alloc(ffq_shard_s* sh) {
  const size_t dim = size_t(1) << sh->l;
  for (int i = 0; i < sh->n_local(); ++i) {
    sh->shards.emplace_back(new DevBuf<double2>());
    sh->shards.back()->alloc(dim);
  }
  if (!sh->group()) {
    sh->sendbuf.alloc(dim);
    sh->recvbuf.alloc(dim);
  }
}

// Support-compacted swap of one rank pair: with valid support bitmaps only the
// supported amplitudes of the two half shards move, as (index, value) lists
// (a UCCSD state fills a few percent of a shard). Returns false when a list
// would exceed a quarter of the shard (dense swap instead). sup0/sup1: the
// pair's bitmaps; s1 == nullptr: NCCL mode (this rank is s0, the partner is
// remote), else both shards are on this device and device copies are the wire.
bool shard_swap_sparse(ffq_shard_s* sh, double2* s0, uint32_t* sup0, int val0, double2* s1, uint32_t* sup1,
                       int val1, int lpos, int partner) {
  ffq_ctx_t ctx = sh->ctx;
  const int l = sh->l;
  const int64_t half = 1LL << (l - 1), cap = half / 2;
  const int64_t words = 1LL << (l - 5);
  const int grid = grid_for(words, ctx->n_sm);
  sh->counters.alloc(4);
  unsigned long long* c = sh->counters.p;
  CK(cudaMemsetAsync(c, 0, 4 * sizeof(unsigned long long), ctx->stream));
  k_swap_count<<<grid, kThreads, 0, ctx->stream>>>(sup0, l, lpos, val0, c);
  unsigned long long n[2] = {0, 0};
  if (s1) {
    k_swap_count<<<grid, kThreads, 0, ctx->stream>>>(sup1, l, lpos, val1, c + 1);
  } else {
    NCK(ncclGroupStart());
    NCK(ncclSend(c, 1, ncclUint64, partner, sh->comm, ctx->stream));
    NCK(ncclRecv(c + 1, 1, ncclUint64, partner, sh->comm, ctx->stream));
    NCK(ncclGroupEnd());
  }
  CK(cudaMemcpyAsync(n, c, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->launches += s1 ? 2 : 1;
  if ((int64_t)n[0] > cap || (int64_t)n[1] > cap) return false;  // both ranks see both counts: same decision
  // values: sendbuf / recvbuf hold 2 * half double2 (two lists of <= cap entries each fit)
  sh->sendidx.alloc((size_t)2 * cap);
  sh->recvidx.alloc((size_t)2 * cap);
  sh->sendbuf.alloc((size_t)2 * cap);
  sh->recvbuf.alloc((size_t)2 * cap);
  double2 *v0 = sh->sendbuf.p, *v1 = sh->sendbuf.p + cap;
  uint32_t *i0 = sh->sendidx.p, *i1 = sh->sendidx.p + cap;
  k_swap_pack_sparse<<<grid, kThreads, 0, ctx->stream>>>(s0, sup0, l, lpos, val0, v0, i0, c + 2);
  if (s1) {
    k_swap_pack_sparse<<<grid, kThreads, 0, ctx->stream>>>(s1, sup1, l, lpos, val1, v1, i1, c + 3);
    // the wire: device copies into the receive buffers
    double2 *r0 = sh->recvbuf.p, *r1 = sh->recvbuf.p + cap;
    uint32_t *j0 = sh->recvidx.p, *j1 = sh->recvidx.p + cap;
    if (n[1]) {
      CK(cudaMemcpyAsync(r0, v1, n[1] * sizeof(double2), cudaMemcpyDeviceToDevice, ctx->stream));
      CK(cudaMemcpyAsync(j0, i1, n[1] * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx->stream));
      k_swap_unpack_sparse<<<grid_for((int64_t)n[1], ctx->n_sm), kThreads, 0, ctx->stream>>>(s0, sup0, lpos, val0, r0, j0,
                                                                                          n[1]);
    }
    if (n[0]) {
      CK(cudaMemcpyAsync(r1, v0, n[0] * sizeof(double2), cudaMemcpyDeviceToDevice, ctx->stream));
      CK(cudaMemcpyAsync(j1, i0, n[0] * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx->stream));
      k_swap_unpack_sparse<<<grid_for((int64_t)n[0], ctx->n_sm), kThreads, 0, ctx->stream>>>(s1, sup1, lpos, val1, r1, j1,
                                                                                          n[0]);
    }
    ctx->launches += 4;
  } else {
    NCK(ncclGroupStart());
    if (n[0]) {
      NCK(ncclSend(v0, (size_t)n[0] * 2, ncclDouble, partner, sh->comm, ctx->stream));
      NCK(ncclSend(i0, (size_t)n[0], ncclUint32, partner, sh->comm, ctx->stream));
    }
    if (n[1]) {
      NCK(ncclRecv(sh->recvbuf.p, (size_t)n[1] * 2, ncclDouble, partner, sh->comm, ctx->stream));
      NCK(ncclRecv(sh->recvidx.p, (size_t)n[1], ncclUint32, partner, sh->comm, ctx->stream));
    }
    NCK(ncclGroupEnd());
    if (n[1])
      k_swap_unpack_sparse<<<grid_for((int64_t)n[1], ctx->n_sm), kThreads, 0, ctx->stream>>>(
          s0, sup0, lpos, val0, sh->recvbuf.p, sh->recvidx.p, n[1]);
    ctx->launches += 2;
  }
  CK(cudaGetLastError());
  return true;
}

// swap physical global position gpos with local lpos on every rank pair;
// sup != nullptr: valid support bitmaps of the local shards ([n_local][2^(l-5)]),
// kept valid by the sparse path; returns false when a dense swap left them stale
bool shard_swap(ffq_shard_s* sh, int gpos, int lpos, uint32_t* sup) {
  ffq_ctx_t ctx = sh->ctx;
  const int j = gpos - sh->l;
  const int64_t half = 1LL << (sh->l - 1);
  const int grid = grid_for(half, ctx->n_sm);
  const int64_t sup_words = sh->l >= 5 ? 1LL << (sh->l - 5) : 0;
  if (sup && sh->group()) {
    bool all = true;
    for (int r = 0; r < sh->R; ++r) {
      if ((r >> j) & 1) continue;
      const int r1 = r ^ (1 << j);
      if (shard_swap_sparse(sh, sh->shards[r]->p, sup + (size_t)r * sup_words, 1, sh->shards[r1]->p,
                            sup + (size_t)r1 * sup_words, 0, lpos, -1)) {
        ++sh->sparse_swaps;
        continue;
      }
      // dense swap of this pair (same kernels as the NCCL transport, a device copy as the wire)
      all = false;
      ++sh->dense_swaps;
      sh->sendbuf.alloc((size_t)2 * half);
      sh->recvbuf.alloc((size_t)2 * half);
      k_swap_pack<<<grid, kThreads, 0, ctx->stream>>>(sh->shards[r]->p, sh->sendbuf.p, sh->l, lpos, 1);
      k_swap_pack<<<grid, kThreads, 0, ctx->stream>>>(sh->shards[r1]->p, sh->sendbuf.p + half, sh->l, lpos, 0);
      CK(cudaMemcpyAsync(sh->recvbuf.p, sh->sendbuf.p + half, sizeof(double2) * half, cudaMemcpyDeviceToDevice,
                         ctx->stream));
      CK(cudaMemcpyAsync(sh->recvbuf.p + half, sh->sendbuf.p, sizeof(double2) * half, cudaMemcpyDeviceToDevice,
                         ctx->stream));
      k_swap_unpack<<<grid, kThreads, 0, ctx->stream>>>(sh->shards[r]->p, sh->recvbuf.p, sh->l, lpos, 1);
      k_swap_unpack<<<grid, kThreads, 0, ctx->stream>>>(sh->shards[r1]->p, sh->recvbuf.p + half, sh->l, lpos, 0);
      CK(cudaGetLastError());
      ctx->launches += 4;
    }
    return all;
  }
  if (sup && !sh->group()) {
    const int bit = (sh->rank >> j) & 1, partner = sh->rank ^ (1 << j);
    if (shard_swap_sparse(sh, sh->shards[0]->p, sup, 1 - bit, nullptr, nullptr, 0, lpos, partner)) {
      ++sh->sparse_swaps;
      return true;
    }
    ++sh->dense_swaps;
  }
  if (sh->group()) {
    // same pack/unpack kernels as the NCCL transport, with a device copy as the wire
    sh->sendbuf.alloc((size_t)2 * half);
    sh->recvbuf.alloc((size_t)2 * half);
    for (int r = 0; r < sh->R; ++r) {
      if ((r >> j) & 1) continue;
      const int r1 = r ^ (1 << j);
      k_swap_pack<<<grid, kThreads, 0, ctx->stream>>>(sh->shards[r]->p, sh->sendbuf.p, sh->l, lpos, 1);
      k_swap_pack<<<grid, kThreads, 0, ctx->stream>>>(sh->shards[r1]->p, sh->sendbuf.p + half, sh->l, lpos, 0);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(sh->recvbuf.p, sh->sendbuf.p + half, sizeof(double2) * half, cudaMemcpyDeviceToDevice,
                         ctx->stream));
      CK(cudaMemcpyAsync(sh->recvbuf.p + half, sh->sendbuf.p, sizeof(double2) * half, cudaMemcpyDeviceToDevice,
                         ctx->stream));
      k_swap_unpack<<<grid, kThreads, 0, ctx->stream>>>(sh->shards[r]->p, sh->recvbuf.p, sh->l, lpos, 1);
      k_swap_unpack<<<grid, kThreads, 0, ctx->stream>>>(sh->shards[r1]->p, sh->recvbuf.p + half, sh->l, lpos, 0);
      CK(cudaGetLastError());
      ctx->launches += 4;
    }
    return false;
  }
  const int bit = (sh->rank >> j) & 1, partner = sh->rank ^ (1 << j);
  k_swap_pack<<<grid, kThreads, 0, ctx->stream>>>(sh->shards[0]->p, sh->sendbuf.p, sh->l, lpos, 1 - bit);
  CK(cudaGetLastError());
  NCK(ncclGroupStart());
  NCK(ncclSend(sh->sendbuf.p, (size_t)half * 2, ncclDouble, partner, sh->comm, ctx->stream));
  NCK(ncclRecv(sh->recvbuf.p, (size_t)half * 2, ncclDouble, partner, sh->comm, ctx->stream));
  NCK(ncclGroupEnd());
  k_swap_unpack<<<grid, kThreads, 0, ctx->stream>>>(sh->shards[0]->p, sh->recvbuf.p, sh->l, lpos, 1 - bit);
  CK(cudaGetLastError());
  ctx->launches += 2;
  return false;
}

double shard_energy(ffq_shard_s* sh, ffq_plan_s* pl, ffq_ham_s* h, uint64_t hf, const double* theta) {
  ffq_ctx_t ctx = sh->ctx;
  const CompiledPlan& cp = pl->cp;
  if (cp.n_qubits != sh->n || h->ch.n_qubits != sh->n)
    throw BadInput("shard: plan / Hamiltonian / shard qubit counts differ", FFQ_EINVAL);
  const int l = sh->l, n_ops = (int)cp.op_kind.size();
  const ShardSchedule S = schedule_shards(cp, sh->g);
  // per-rank rotation coefficients; string ops fold the global Z sign into sin
  std::vector<double2> cs((size_t)sh->n_local() * std::max(1, n_ops));
  std::vector<uint64_t> pbits(cp.pair_bits.size());
  std::vector<uint32_t> plow(cp.pair_bits.size(), 0u);
  std::vector<FusedDesc> phys(cp.fused.size());
  std::vector<int> perm = S.init_perm;
  std::vector<std::vector<int>> op_perm(n_ops);
  for (const auto& st : S.steps) {
    if (st.kind == 0) {
      int qa = -1, qb = -1;
      for (int q = 0; q < sh->n; ++q) {
        if (perm[q] == st.gpos) qa = q;
        if (perm[q] == st.lpos) qb = q;
      }
      std::swap(perm[qa], perm[qb]);
    } else {
      op_perm[st.op] = perm;
    }
  }
  for (int op = 0; op < n_ops; ++op) {
    const double phi = theta[cp.op_gen[op]] * cp.op_cfac[op];
    if (cp.op_kind[op] == 0) {
      const FusedDesc& d = cp.fused[cp.op_idx[op]];
      phys[cp.op_idx[op]] = physical_fused(d, op_perm[op]);
      for (int p = 0; p < d.npair; ++p) {
        pbits[d.pair_off + p] = permute_mask(cp.pair_bits[d.pair_off + p], op_perm[op]);
        plow[d.pair_off + p] = low_pattern_mask(phys[cp.op_idx[op]].x, pbits[d.pair_off + p]);
      }
    }
    for (int i = 0; i < sh->n_local(); ++i) {
      // Z on global qubits is a per-rank sign, folded into sin (string ops: the
      // string's z; fused ops: the outside-Z mask of the generator)
      const uint64_t zp = cp.op_kind[op] == 1 ? permute_mask(cp.str_z[cp.op_idx[op]], op_perm[op])
                                              : phys[cp.op_idx[op]].zout;
      const double sg = (__builtin_popcountll(((uint64_t)sh->rank_of(i) << l) & zp) & 1) ? -1.0 : 1.0;
      cs[(size_t)i * n_ops + op] = make_double2(std::cos(phi), std::sin(phi) * cp.op_sscale[op] * sg);
    }
  }
  sh->cs.upload(cs, ctx->stream);
  sh->pbits.upload(pbits, ctx->stream);
  sh->plow.upload(plow, ctx->stream);
  // |HF> on its owner rank
  const uint64_t hf_phys = permute_mask(hf, S.init_perm);
  for (int i = 0; i < sh->n_local(); ++i) {
    CK(cudaMemsetAsync(sh->shards[i]->p, 0, sizeof(double2) << l, ctx->stream));
    if ((uint64_t)sh->rank_of(i) == (hf_phys >> l)) {
      const double2 one = make_double2(1.0, 0.0);
      CK(cudaMemcpyAsync(sh->shards[i]->p + (hf_phys & ((1ULL << l) - 1)), &one, sizeof(one),
                         cudaMemcpyHostToDevice, ctx->stream));
    }
  }
  // support bitmaps of the local shards (bit k % 32 of word k / 32: amplitude k may be
  // non-zero), kept by the support-tracked generator passes and rebuilt from the
  // data after a swap or a dense string pass
  const bool track = use_support(ctx, l);
  const int64_t sup_words = l >= 5 ? 1LL << (l - 5) : 0;
  bool stale = false;
  auto rebuild = [&] {
    for (int i = 0; i < sh->n_local(); ++i)
      launch_support_from_state(ctx, sh->shards[i]->p, sh->sup_own.p + (size_t)i * sup_words, l, 1);
    stale = false;
  };
  if (track) {
    sh->sup_own.alloc((size_t)sup_words * sh->n_local());
    rebuild();  // |HF> only
  }
  sh->last_swaps = 0;
  for (const auto& st : S.steps) {
    if (st.kind == 0) {
      // (the sparse swap needs valid bitmaps and keeps them valid)
      if (track && stale) rebuild();
      if (!shard_swap(sh, st.gpos, st.lpos, track ? sh->sup_own.p : nullptr)) stale = true;
      ++sh->last_swaps;
      continue;
    }
    const int op = st.op;
    for (int i = 0; i < sh->n_local(); ++i) {
      const double2* csr = sh->cs.p + (size_t)i * n_ops;
      if (cp.op_kind[op] == 0) {
        const FusedDesc& d = phys[cp.op_idx[op]];
        if (track) {  // support-tracked pass (the global Z sign is in csr)
          if (stale && i == 0) rebuild();
          const int64_t work = (int64_t)d.npair << (l - 5 - d.whi);
          k_fused_gen_support<<<grid_for(work, ctx->n_sm), kThreads, 0, ctx->stream>>>(
              sh->shards[i]->p, sh->sup_own.p + (size_t)i * sup_words, l, d, sh->pbits.p, sh->plow.p, pl->pair_f.p,
              csr, n_ops, op, 1LL << l);
          CK(cudaGetLastError());
          ctx->launches++;
          continue;
        }
        const bool vec = !(d.x & 1ULL) && (l - d.w) >= 1;
        const int64_t work = ((int64_t)d.npair << (l - d.w)) >> (vec ? 1 : 0);
        if (vec)
          k_fused_gen<true><<<grid_for(work, ctx->n_sm), kThreads, 0, ctx->stream>>>(
              sh->shards[i]->p, l, d, sh->pbits.p, pl->pair_f.p, csr, n_ops, op, 0);
        else
          k_fused_gen<false><<<grid_for(work, ctx->n_sm), kThreads, 0, ctx->stream>>>(
              sh->shards[i]->p, l, d, sh->pbits.p, pl->pair_f.p, csr, n_ops, op, 0);
        CK(cudaGetLastError());
        ctx->launches++;
      } else {
        stale = true;
        const int si = cp.op_idx[op];
        const uint64_t lm = (1ULL << l) - 1ULL;
        const uint64_t xp = permute_mask(cp.str_x[si], op_perm[op]);
        const uint64_t zp = permute_mask(cp.str_z[si], op_perm[op]) & lm;
        launch_string(ctx, sh->shards[i]->p, l, 1, xp, zp, cp.str_ny[si], csr, n_ops, op);
      }
    }
  }
  sh->perm = S.final_perm;
  // physical Hamiltonian for the final permutation (cached)
  if (sh->ham_key != h->uid || sh->ham_perm != S.final_perm || !sh->hphys) {
    std::vector<uint64_t> x(h->raw_x.size()), z(h->raw_z.size());
    for (size_t t = 0; t < x.size(); ++t) {
      x[t] = permute_mask(h->raw_x[t], S.final_perm);
      z[t] = permute_mask(h->raw_z[t], S.final_perm);
    }
    auto hp = std::make_unique<ffq_ham_s>();
    hp->ctx = ctx;
    hp->ch = compile_ham(sh->n, (int64_t)x.size(), x.data(), z.data(), h->raw_re.data(), h->raw_im.data());
    hp->ch.item_chunk = std::max<int64_t>(kItemChunk, (1LL << (l - 1)) / 256);
    const auto& ch = hp->ch;
    hp->groups.upload(ch.groups, ctx->stream);
    hp->act_bits.upload(ch.act_bits, ctx->stream);
    hp->cls_z.upload(ch.cls_z, ctx->stream);
    std::vector<double2> f(ch.cls_f.size() / 2);
    for (size_t i = 0; i < f.size(); ++i) f[i] = make_double2(ch.cls_f[2 * i], ch.cls_f[2 * i + 1]);
    hp->cls_f.upload(f, ctx->stream);
    // one-term groups in generic mode (|X| > 6) leave the item list: they run
    // batched per out-of-shard flip pattern, every local member enumerated
    // (weight 1, full z: the folded pair-once weight 2 and the cleared pairing
    // bit of the generic class are undone from the raw term)
    std::map<uint64_t, std::map<uint64_t, double>> byx;
    for (size_t t = 0; t < x.size(); ++t) byx[x[t]][z[t]] += h->raw_re[t];
    std::map<uint32_t, std::vector<ShardTerm>> multi;  // hG -> terms, ascending X
    std::set<uint64_t> multi_x;
    for (const auto& gx : byx) {
      if (l < 5 || __builtin_popcountll(gx.first) <= kMaxTableBits) continue;  // (bitmap words need 32 amplitudes)
      int live = 0;
      uint64_t zz = 0;
      double cc = 0.0;
      for (const auto& kv : gx.second)
        if (kv.second != 0.0) { ++live; zz = kv.first; cc = kv.second; }
      if (live != 1) continue;
      const int ny = __builtin_popcountll(gx.first & zz) & 3;
      const double2 f = make_double2(ny == 0 ? cc : ny == 2 ? -cc : 0.0, ny == 1 ? cc : ny == 3 ? -cc : 0.0);
      multi[(uint32_t)(gx.first >> l)].push_back({gx.first & ((1ULL << l) - 1ULL), zz, f});
      multi_x.insert(gx.first);
    }
    {
      std::vector<ShardTerm> mt;
      std::vector<int2> mb;
      sh->mbuckets.clear();
      for (const auto& kv : multi) {
        ffq_shard_s::MultiBucket bk{kv.first, (int)mb.size(), 0};
        for (size_t t0 = 0; t0 < kv.second.size(); t0 += 16) {
          mb.push_back(make_int2((int)(mt.size() + t0), (int)std::min<size_t>(16, kv.second.size() - t0)));
          ++bk.n_batches;
        }
        mt.insert(mt.end(), kv.second.begin(), kv.second.end());
        sh->mbuckets.push_back(bk);
      }
      sh->mterms.upload(mt, ctx->stream);
      sh->mbatches.upload(mb, ctx->stream);
      const int64_t words = l >= 5 ? 1LL << (l - 5) : 1;
      sh->mchunk = std::max<int64_t>(kItemChunk, words / 512);
      sh->mchunks = (words + sh->mchunk - 1) / sh->mchunk;
    }
    // items over the local index space (the global part of X picks the partner)
    std::vector<int32_t> ig, ip;
    std::vector<int64_t> iu;
    for (size_t gi = 0; gi < ch.groups.size(); ++gi) {
      const auto& d = ch.groups[gi];
      if (multi_x.count(d.x)) continue;
      uint64_t Q = 0;  // inserted positions (see k_expect_shard)
      for (int i = 0; i < d.w; ++i) Q |= 1ULL << d.q[i];
      const int wl = __builtin_popcountll(Q & ((1ULL << l) - 1ULL));
      const int64_t U = 1LL << (l - wl);
      for (int p = 0; p < d.nact; ++p)
        for (int64_t u0 = 0; u0 < U; u0 += hp->ch.item_chunk) {
          ig.push_back((int32_t)gi);
          ip.push_back(p);
          iu.push_back(u0);
        }
    }
    hp->ch.item_g = ig;
    hp->ch.item_p = ip;
    hp->ch.item_u0 = iu;
    hp->item_g.upload(ig, ctx->stream);
    hp->item_p.upload(ip, ctx->stream);
    hp->item_u0.upload(iu, ctx->stream);
    sh->hphys = std::move(hp);
    sh->ham_key = h->uid;
    sh->ham_perm = S.final_perm;
  }
  const ffq_ham_s* hp = sh->hphys.get();
  const int64_t items_old = (int64_t)hp->ch.item_g.size();
  int64_t n_mbatches = 0;
  for (const auto& bk : sh->mbuckets) n_mbatches += bk.n_batches;
  const int64_t items = items_old + n_mbatches * sh->mchunks;  // partial slots per local shard
  sh->partial.alloc((size_t)std::max<int64_t>(1, items) * sh->n_local());
  sh->eloc.alloc(std::max<size_t>(2 * (size_t)sh->n_local(), (size_t)sh->R + 1));
  if (items > 0) CK(cudaMemsetAsync(sh->partial.p, 0, sizeof(double2) * items * sh->n_local(), ctx->stream));
  // support bitmaps of the local shards for the batched one-term groups
  if (!sh->mbuckets.empty()) {
    sh->sup_own.alloc((size_t)sup_words * sh->n_local());
    if (!sh->group()) sh->sup_partner.alloc((size_t)sup_words);
    if (!track || stale) rebuild();  // (tracked bitmaps are conservative supersets: fine)
  }
  // buckets of one out-of-shard flip pattern hG, ascending: the items sharing hG
  // are contiguous (groups sorted by X), the batched one-term groups per bucket
  int64_t i0 = 0;
  size_t mb = 0;
  while (i0 < items_old || mb < sh->mbuckets.size()) {
    const uint32_t h_old = i0 < items_old ? (uint32_t)(hp->ch.groups[hp->ch.item_g[i0]].x >> l) : 0xFFFFFFFFu;
    const uint32_t h_multi = mb < sh->mbuckets.size() ? sh->mbuckets[mb].hG : 0xFFFFFFFFu;
    const uint32_t hG = std::min(h_old, h_multi);
    int64_t i1 = i0;
    while (i1 < items_old && (uint32_t)(hp->ch.groups[hp->ch.item_g[i1]].x >> l) == hG) ++i1;
    const double2* partner_nccl = nullptr;
    if (!sh->group() && hG != 0) {
      const int partner = sh->rank ^ (int)hG;
      NCK(ncclGroupStart());
      NCK(ncclSend(sh->shards[0]->p, (size_t)2 << l, ncclDouble, partner, sh->comm, ctx->stream));
      NCK(ncclRecv(sh->recvbuf.p, (size_t)2 << l, ncclDouble, partner, sh->comm, ctx->stream));
      NCK(ncclGroupEnd());
      partner_nccl = sh->recvbuf.p;
      if (h_multi == hG) launch_support_from_state(ctx, sh->recvbuf.p, sh->sup_partner.p, l, 1);
    }
    for (int i = 0; i < sh->n_local(); ++i) {
      const int r = sh->rank_of(i);
      const double2* partner = hG == 0 ? sh->shards[i]->p
                               : sh->group() ? sh->shards[r ^ (int)hG]->p
                                             : partner_nccl;
      const uint32_t* partner_sup = hG == 0 ? sh->sup_own.p + (size_t)i * sup_words
                                    : sh->group() ? sh->sup_own.p + (size_t)(r ^ (int)hG) * sup_words
                                                  : sh->sup_partner.p;
      if (i1 > i0) {
        k_expect_shard<kThreads><<<(unsigned)(i1 - i0), kThreads, 0, ctx->stream>>>(
            sh->shards[i]->p, partner, l, (uint32_t)r, hp->dev(), i0, sh->partial.p + (size_t)i * items);
        CK(cudaGetLastError());
        ctx->launches++;
      }
      if (h_multi == hG) {
        const auto& bk = sh->mbuckets[mb];
        const int64_t slot0 = items_old + (int64_t)bk.batch0 * sh->mchunks;
        k_expect_shard_multi<kThreads><<<dim3((unsigned)sh->mchunks, (unsigned)bk.n_batches), kThreads, 0, ctx->stream>>>(
            sh->shards[i]->p, partner, sh->sup_own.p + (size_t)i * sup_words, partner_sup, l, (uint32_t)r,
            sh->mterms.p, sh->mbatches.p, bk.batch0, sh->mchunk, slot0,
            sh->partial.p + (size_t)i * items);
        CK(cudaGetLastError());
        ctx->launches++;
      }
    }
    i0 = i1;
    if (h_multi == hG) ++mb;
  }
  for (int i = 0; i < sh->n_local(); ++i) {
    k_reduce_partials<kThreads><<<1, kThreads, 0, ctx->stream>>>(sh->partial.p + (size_t)i * std::max<int64_t>(1, items),
                                                                 std::max<int64_t>(1, items),
                                                                 sh->eloc.p + i, nullptr);
    CK(cudaGetLastError());
    ctx->launches++;
  }
  std::vector<double> e_rank((size_t)sh->R, 0.0);
  if (sh->group()) {
    CK(cudaMemcpyAsync(e_rank.data(), sh->eloc.p, sizeof(double) * sh->R, cudaMemcpyDeviceToHost, ctx->stream));
  } else {
    NCK(ncclAllGather(sh->eloc.p, sh->eloc.p + 1, 1, ncclDouble, sh->comm, ctx->stream));
    CK(cudaMemcpyAsync(e_rank.data(), sh->eloc.p + 1, sizeof(double) * sh->R, cudaMemcpyDeviceToHost,
                       ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  double e = 0.0;
  for (double v : e_rank) e += v;  // rank order: deterministic
  return e;
}

}  // namespace

extern "C" {

int ffq_shard_create(ffq_ctx_t ctx, int n_qubits, int n_global, ffq_shard_t* out) {
  if (!ctx || !out || n_global < 0 || n_global > 6 || n_qubits - n_global < 2 || n_qubits > 40)
    return fail(ctx, FFQ_EINVAL, "ffq_shard_create: need 0 <= n_global <= 6 and n_qubits - n_global >= 2");
  *out = nullptr;
  return guarded_shard(ctx, [&] {
    auto sh = std::make_unique<ffq_shard_s>();
    sh->ctx = ctx;
    sh->n = n_qubits;
    sh->g = n_global;
    sh->l = n_qubits - n_global;
    sh->R = 1 << n_global;
    shard_alloc(sh.get());
    *out = sh.release();
    return FFQ_OK;
  });
}

int ffq_nccl_unique_id(void* id128) {
  if (!id128) return fail(nullptr, FFQ_EINVAL, "null argument");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, FFQ_ENCCL, ncclGetErrorString(r));
  std::memcpy(id128, &id, sizeof(id));
  return FFQ_OK;
}

int ffq_shard_create_nccl(ffq_ctx_t ctx, int n_qubits, int n_global, int rank, const void* id128,
                          ffq_shard_t* out) {
  if (!ctx || !out || !id128 || n_global < 0 || n_global > 6 || n_qubits - n_global < 2 || rank < 0 ||
      rank >= (1 << n_global))
    return fail(ctx, FFQ_EINVAL, "ffq_shard_create_nccl: invalid argument");
  *out = nullptr;
  return guarded_shard(ctx, [&] {
    auto sh = std::make_unique<ffq_shard_s>();
    sh->ctx = ctx;
    sh->n = n_qubits;
    sh->g = n_global;
    sh->l = n_qubits - n_global;
    sh->R = 1 << n_global;
    sh->rank = rank;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    NCK(ncclCommInitRank(&sh->comm, sh->R, id, rank));
    shard_alloc(sh.get());
    *out = sh.release();
    return FFQ_OK;
  });
}

int ffq_shard_destroy(ffq_shard_t sh) {
  if (sh) {
    cudaSetDevice(sh->ctx->device);
    cudaStreamSynchronize(sh->ctx->stream);
    delete sh;
  }
  return FFQ_OK;
}

int ffq_shard_energy(ffq_shard_t sh, ffq_plan_t plan, ffq_ham_t ham, uint64_t hf_bits, const double* theta,
                     double* e_out) {
  if (!sh || !plan || !ham || !e_out || (!theta && plan->cp.n_gen > 0))
    return fail(sh ? sh->ctx : nullptr, FFQ_EINVAL, "ffq_shard_energy: null argument");
  return guarded_shard(sh->ctx, [&] {
    *e_out = shard_energy(sh, plan, ham, hf_bits, theta);
    return FFQ_OK;
  });
}

int ffq_shard_download(ffq_shard_t sh, double* psi) {
  if (!sh || !psi) return fail(sh ? sh->ctx : nullptr, FFQ_EINVAL, "null argument");
  if (!sh->group()) return fail(sh->ctx, FFQ_EINVAL, "ffq_shard_download: group mode only");
  return guarded_shard(sh->ctx, [&] {
    const size_t dim = size_t(1) << sh->l;
    std::vector<double2> host(dim);
    std::vector<int> inv(sh->n);
    const std::vector<int>& perm = sh->perm.empty() ? std::vector<int>() : sh->perm;
    for (int q = 0; q < sh->n; ++q) inv[perm.empty() ? q : perm[q]] = q;
    for (int r = 0; r < sh->R; ++r) {
      CK(cudaMemcpyAsync(host.data(), sh->shards[r]->p, sizeof(double2) * dim, cudaMemcpyDeviceToHost,
                         sh->ctx->stream));
      CK(cudaStreamSynchronize(sh->ctx->stream));
      for (size_t k = 0; k < dim; ++k) {
        const uint64_t phys = ((uint64_t)r << sh->l) | k;
        uint64_t logical = 0;
        for (int pq = 0; pq < sh->n; ++pq)
          if ((phys >> pq) & 1ULL) logical |= 1ULL << inv[pq];
        psi[2 * logical] = host[k].x;
        psi[2 * logical + 1] = host[k].y;
      }
    }
    return FFQ_OK;
  });
}

int ffq_shard_info(ffq_shard_t sh, int* last_swaps, int* perm_out) {
  if (!sh) return fail(nullptr, FFQ_EINVAL, "null shard");
  if (last_swaps) *last_swaps = sh->last_swaps;
  if (perm_out)
    for (int q = 0; q < sh->n; ++q) perm_out[q] = sh->perm.empty() ? q : sh->perm[q];
  return FFQ_OK;
}

int ffq_shard_schedule(int n_qubits, int n_global, int n_gen, const int64_t* term_off, const uint64_t* x,
                       const uint64_t* z, const double* c_re, const double* c_im, int* init_perm,
                       int* final_perm, int* n_swaps, int* n_steps) {
  return ffq_shard_schedule_steps(n_qubits, n_global, n_gen, term_off, x, z, c_re, c_im, init_perm, final_perm,
                                  n_swaps, n_steps, nullptr, 0);
}

int ffq_shard_schedule_steps(int n_qubits, int n_global, int n_gen, const int64_t* term_off, const uint64_t* x,
                             const uint64_t* z, const double* c_re, const double* c_im, int* init_perm,
                             int* final_perm, int* n_swaps, int* n_steps, int* steps, int max_steps) {
  return guarded(nullptr, [&] {
    const CompiledPlan P = compile_plan(n_qubits, n_gen, term_off, x, z, c_re, c_im);
    const ShardSchedule S = schedule_shards(P, n_global);
    for (int q = 0; q < n_qubits; ++q) {
      if (init_perm) init_perm[q] = S.init_perm[q];
      if (final_perm) final_perm[q] = S.final_perm[q];
    }
    if (n_swaps) *n_swaps = S.n_swaps();
    if (n_steps) *n_steps = (int)S.steps.size();
    if (steps) {
      if ((int)S.steps.size() > max_steps) throw BadInput("ffq_shard_schedule_steps: steps buffer too small", FFQ_EINVAL);
      for (size_t i = 0; i < S.steps.size(); ++i) {
        // kind, gpos, lpos, generator index (plan column) of the op
        steps[4 * i] = S.steps[i].kind;
        steps[4 * i + 1] = S.steps[i].gpos;
        steps[4 * i + 2] = S.steps[i].lpos;
        steps[4 * i + 3] = S.steps[i].kind ? P.op_gen[S.steps[i].op] : -1;
      }
    }
    return FFQ_OK;
  });
}

}  // extern "C"
