// ffq_krylov.inl -- lanczos_ground and energy_exact (
// SURVEY.md 8f2). Included at the end of ffq_capi.cu.
//
// Both work on a closure basis (compile_krylov) with the Hamiltonian and the
// generator matrix as device CSR; every matrix-vector product is the
// k_csr_matvec kernel, the small host-side recurrences (Lanczos with full
// reorthogonalisation, Taylor series) are O(basis) vector work.

namespace {

struct DeviceCsr {
  int64_t rows = 0;
  DevBuf<int64_t> rp;
  DevBuf<uint32_t> col;
  DevBuf<double> re, im;
  DevBuf<int32_t> gen;
  bool has_gen = false;
};

void upload_csr(ffq_ctx_t ctx, DeviceCsr& d, const std::vector<int64_t>& rp, const std::vector<uint32_t>& col,
                const std::vector<double>& re, const std::vector<double>& im, const std::vector<int32_t>* gen) {
  d.rows = (int64_t)rp.size() - 1;
  d.rp.upload(rp, ctx->stream);
  d.col.upload(col, ctx->stream);
  d.re.upload(re, ctx->stream);
  d.im.upload(im, ctx->stream);
  d.has_gen = gen != nullptr;
  if (gen) d.gen.upload(*gen, ctx->stream);
}

using cvec = std::vector<std::complex<double>>;

// y = M x on the device (x, y host vectors of length rows)
void csr_apply(ffq_ctx_t ctx, const DeviceCsr& M, const double* theta_dev, DevBuf<double2>& xd,
               DevBuf<double2>& yd, const cvec& x, cvec& y) {
  const size_t n = (size_t)M.rows;
  xd.alloc(n);
  yd.alloc(n);
  CK(cudaMemcpyAsync(xd.p, x.data(), n * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
  k_csr_matvec<<<grid_for((int64_t)n * 32, ctx->n_sm), kThreads, 0, ctx->stream>>>(
      M.rows, M.rp.p, M.col.p, M.re.p, M.im.p, M.has_gen ? M.gen.p : nullptr, theta_dev, xd.p, yd.p);
  CK(cudaGetLastError());
  ctx->launches++;
  y.resize(n);
  CK(cudaMemcpyAsync(y.data(), yd.p, n * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
}

std::complex<double> vdot(const cvec& a, const cvec& b) {
  std::complex<double> s(0, 0);
  for (size_t i = 0; i < a.size(); ++i) s += std::conj(a[i]) * b[i];
  return s;
}

// smallest eigenvalue of the symmetric tridiagonal (a, b) by Sturm bisection
double tridiag_min_eig(const std::vector<double>& a, const std::vector<double>& b) {
  const size_t k = a.size();
  double lo = 1e300, hi = -1e300;
  for (size_t i = 0; i < k; ++i) {
    const double r = (i > 0 ? std::abs(b[i - 1]) : 0.0) + (i + 1 < k ? std::abs(b[i]) : 0.0);
    lo = std::min(lo, a[i] - r);
    hi = std::max(hi, a[i] + r);
  }
  auto count_below = [&](double x) {  // eigenvalues < x
    int c = 0;
    double q = a[0] - x;
    if (q < 0) ++c;
    for (size_t i = 1; i < k; ++i) {
      q = a[i] - x - b[i - 1] * b[i - 1] / (q != 0.0 ? q : 1e-300);
      if (q < 0) ++c;
    }
    return c;
  };
  for (int it = 0; it < 200 && hi - lo > 1e-15 * std::max(1.0, std::abs(lo)); ++it) {
    const double mid = 0.5 * (lo + hi);
    if (count_below(mid) >= 1) hi = mid; else lo = mid;
  }
  return 0.5 * (lo + hi);
}

}  // namespace

extern "C" {

int ffq_lanczos_ground(ffq_ctx_t ctx, ffq_ham_t ham, uint64_t hf_bits, double tol, int max_iter, double* e0,
                       int* iters, int* dim) {
  if (!ctx || !ham || !e0) return fail(ctx, FFQ_EINVAL, "ffq_lanczos_ground: null argument");
  return guarded(ctx, [&] {
    const int n = ham->ch.n_qubits;
    if (n < 64 && (hf_bits >> n)) throw BadInput("hf_bits exceeds n_qubits", FFQ_EINVAL);
    const KrylovSpace K = compile_krylov(ham->ch, nullptr, hf_bits, 1u << 22, true);
    if (!K.ok) throw BadInput("lanczos_ground: " + K.why, FFQ_EINVAL);
    DeviceCsr Hm;
    upload_csr(ctx, Hm, K.h_row, K.h_col, K.h_re, K.h_im, nullptr);
    const size_t N = K.basis.size();
    DevBuf<double2> xd, yd;
    std::vector<cvec> V;
    cvec v(N, {0.0, 0.0}), w;
    v[K.hf_idx] = 1.0;
    std::vector<double> al, be;
    double e_prev = 0.0, e = 0.0;
    int k = 0;
    const int kmax = std::max(1, std::min<int>(max_iter > 0 ? max_iter : 500, (int)N));
    for (; k < kmax; ++k) {
      V.push_back(v);
      csr_apply(ctx, Hm, nullptr, xd, yd, v, w);
      const double a = vdot(v, w).real();
      al.push_back(a);
      for (size_t i = 0; i < N; ++i) w[i] -= a * v[i];
      if (k > 0)
        for (size_t i = 0; i < N; ++i) w[i] -= be.back() * V[k - 1][i];
      for (int pass = 0; pass < 2; ++pass)  // full reorthogonalisation
        for (const auto& u : V) {
          const std::complex<double> c = vdot(u, w);
          for (size_t i = 0; i < N; ++i) w[i] -= c * u[i];
        }
      e = tridiag_min_eig(al, be);
      double b = 0.0;
      for (auto& x : w) b += std::norm(x);
      b = std::sqrt(b);
      if ((k > 1 && std::abs(e - e_prev) <= tol) || b < 1e-12) { ++k; break; }
      e_prev = e;
      be.push_back(b);
      for (size_t i = 0; i < N; ++i) v[i] = w[i] / b;
    }
    *e0 = e;
    if (iters) *iters = k;
    if (dim) *dim = (int)N;
    return FFQ_OK;
  });
}

int ffq_energy_exact(ffq_ctx_t ctx, ffq_plan_t plan, ffq_ham_t ham, uint64_t hf_bits, const double* theta,
                     double tol, double* e_out) {
  if (!ctx || !plan || !ham || !e_out || (!theta && plan->cp.n_gen > 0))
    return fail(ctx, FFQ_EINVAL, "ffq_energy_exact: null argument");
  return guarded(ctx, [&] {
    if (plan->cp.n_qubits != ham->ch.n_qubits) throw BadInput("plan and Hamiltonian qubit counts differ", FFQ_EINVAL);
    const KrylovSpace K = compile_krylov(ham->ch, &plan->cp, hf_bits, 1u << 22, false);
    if (!K.ok) throw BadInput("energy_exact: " + K.why, FFQ_EINVAL);
    DeviceCsr Hm, Am;
    upload_csr(ctx, Hm, K.h_row, K.h_col, K.h_re, K.h_im, nullptr);
    upload_csr(ctx, Am, K.a_row, K.a_col, K.a_re, K.a_im, &K.a_gen);
    DevBuf<double> th;
    th.alloc(std::max(1, plan->cp.n_gen));
    if (plan->cp.n_gen)
      CK(cudaMemcpyAsync(th.p, theta, sizeof(double) * plan->cp.n_gen, cudaMemcpyHostToDevice, ctx->stream));
    const size_t N = K.basis.size();
    DevBuf<double2> xd, yd;
    cvec psi(N, {0.0, 0.0}), term(N, {0.0, 0.0}), nxt;
    term[K.hf_idx] = 1.0;
    psi = term;
    // e^{A}|hf> = sum_k A^k |hf> / k!, stopped when the term norm is below tol
    const double eps = tol > 0 ? tol : 1e-12;
    int k = 1;
    for (; k <= 200; ++k) {
      csr_apply(ctx, Am, th.p, xd, yd, term, nxt);
      double nn = 0.0;
      for (size_t i = 0; i < N; ++i) {
        term[i] = nxt[i] / (double)k;
        psi[i] += term[i];
        nn += std::norm(term[i]);
      }
      if (std::sqrt(nn) <= eps * 1e-2) break;
    }
    if (k > 200) throw BadInput("energy_exact: Taylor series did not converge in 200 terms", FFQ_EINVAL);
    cvec hpsi;
    csr_apply(ctx, Hm, nullptr, xd, yd, psi, hpsi);
    const std::complex<double> e = vdot(psi, hpsi);
    if (std::abs(e.imag()) > 1e-10) throw BadInput("energy_exact: imaginary residue", FFQ_ENONHERMITIAN);
    *e_out = e.real();
    return FFQ_OK;
  });
}

}  // extern "C"
