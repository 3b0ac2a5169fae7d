// ffq_multi.inl -- the C-ABI's multi-GPU front end for the independent-unit
// workloads (BASELINE configs 2-4): batched theta rows and FMO
// fragments shard over the devices of one node with no data-path collective.
// One context per device, one host thread per device per call; a row's
// energy does not depend on which device or batch computes it (the sector
// programs are per-row deterministic), so every split gives the bits of the
// one-device call. Included by ffq_capi.cu.
#include <thread>

struct ffq_multi_s {
  std::vector<ffq_ctx_t> ctx;                                       // one per device
  std::vector<std::vector<std::pair<ffq_plan_t, ffq_ham_t>>> probs;  // [problem][device]
  std::vector<int> n_qubits, n_gen;
  std::vector<double> cost;                                          // per evaluation (fragment_cost units)
  std::string err;
};

namespace {

int multi_fail(ffq_multi_t m, int code, const std::string& msg) {
  if (m) m->err = msg;
  return fail(nullptr, code, msg);
}

// run f(d) for every device d on its own host thread; the first failure wins
template <class F>
int on_devices(ffq_multi_t m, const std::vector<int>& devs, F&& f) {
  std::vector<int> rc(devs.size(), FFQ_OK);
  std::vector<std::thread> th;
  for (size_t k = 0; k < devs.size(); ++k) th.emplace_back([&, k] { rc[k] = f(devs[k]); });
  for (auto& t : th) t.join();
  for (size_t k = 0; k < devs.size(); ++k)
    if (rc[k] != FFQ_OK) {
      m->err = std::string("device ") + std::to_string(devs[k]) + ": " + ffq_last_error(m->ctx[devs[k]]);
      return rc[k];
    }
  return FFQ_OK;
}

std::vector<int> all_devices(ffq_multi_t m) {
  std::vector<int> d(m->ctx.size());
  for (size_t k = 0; k < d.size(); ++k) d[k] = (int)k;
  return d;
}

}  // namespace

extern "C" {

int ffq_multi_create(const int* devices, int n_dev, ffq_multi_t* out) {
  if (!out || !devices || n_dev < 1) return fail(nullptr, FFQ_EINVAL, "ffq_multi_create: invalid argument");
  *out = nullptr;
  auto* m = new ffq_multi_s();
  for (int k = 0; k < n_dev; ++k) {
    for (int q = 0; q < k; ++q)
      if (devices[q] == devices[k]) {
        ffq_multi_destroy(m);
        return fail(nullptr, FFQ_EINVAL, "ffq_multi_create: device listed twice");
      }
    ffq_ctx_t c = nullptr;
    const int rc = ffq_ctx_create(devices[k], &c);
    if (rc != FFQ_OK) {
      ffq_multi_destroy(m);
      return rc;
    }
    m->ctx.push_back(c);
  }
  *out = m;
  return FFQ_OK;
}

int ffq_multi_destroy(ffq_multi_t m) {
  if (!m) return FFQ_OK;
  for (auto& per : m->probs)
    for (auto& ph : per) {
      ffq_plan_destroy(ph.first);
      ffq_ham_destroy(ph.second);
    }
  for (ffq_ctx_t c : m->ctx) ffq_ctx_destroy(c);
  delete m;
  return FFQ_OK;
}

int ffq_multi_device_count(ffq_multi_t m, int* n) {
  if (!m || !n) return fail(nullptr, FFQ_EINVAL, "ffq_multi_device_count: invalid argument");
  *n = (int)m->ctx.size();
  return FFQ_OK;
}

const char* ffq_multi_last_error(ffq_multi_t m) { return m ? m->err.c_str() : ffq_last_error(nullptr); }

int ffq_multi_problem_upload(ffq_multi_t m, int n_qubits, int n_gen, const int64_t* term_off, const uint64_t* px,
                             const uint64_t* pz, const double* pc_re, const double* pc_im, int64_t n_terms,
                             const uint64_t* hx, const uint64_t* hz, const double* hc_re, const double* hc_im,
                             int* problem_out) {
  if (!m || !problem_out) return fail(nullptr, FFQ_EINVAL, "ffq_multi_problem_upload: invalid argument");
  std::vector<std::pair<ffq_plan_t, ffq_ham_t>> per(m->ctx.size(), {nullptr, nullptr});
  const int rc = on_devices(m, all_devices(m), [&](int d) {
    int r = ffq_plan_upload(m->ctx[d], n_qubits, n_gen, term_off, px, pz, pc_re, pc_im, &per[d].first);
    if (r == FFQ_OK) r = ffq_ham_upload(m->ctx[d], n_qubits, n_terms, hx, hz, hc_re, hc_im, &per[d].second);
    return r;
  });
  if (rc != FFQ_OK) {
    for (auto& ph : per) {
      if (ph.first) ffq_plan_destroy(ph.first);
      if (ph.second) ffq_ham_destroy(ph.second);
    }
    return rc;
  }
  int n_groups = 0;
  int64_t nt = 0, ncls = 0;
  ffq_ham_info(per[0].second, &n_groups, &nt, &ncls);
  *problem_out = (int)m->probs.size();
  m->probs.push_back(std::move(per));
  m->n_qubits.push_back(n_qubits);
  m->n_gen.push_back(n_gen);
  // cost of one evaluation ~ 2^n x (generators + flip-mask groups) (fragment_cost)
  m->cost.push_back(std::ldexp(1.0, n_qubits) * (double)(n_gen + n_groups));
  return FFQ_OK;
}

int ffq_multi_energy_batch(ffq_multi_t m, int problem, uint64_t hf_bits, int batch, const double* theta,
                           double* e_out) {
  if (!m || problem < 0 || problem >= (int)m->probs.size() || batch < 0 || (batch > 0 && (!theta || !e_out)))
    return multi_fail(m, FFQ_EINVAL, "ffq_multi_energy_batch: invalid argument");
  if (batch == 0) return FFQ_OK;
  const int D = (int)m->ctx.size(), ng = m->n_gen[problem];
  // contiguous row blocks, sizes differing by at most one (dist.row_range)
  auto range = [&](int d) {
    const int base = batch / D, extra = batch % D;
    const int lo = d * base + std::min(d, extra);
    return std::make_pair(lo, lo + base + (d < extra ? 1 : 0));
  };
  return on_devices(m, all_devices(m), [&](int d) {
    const auto r = range(d);
    if (r.second == r.first) return (int)FFQ_OK;
    const auto& ph = m->probs[problem][d];
    return ffq_energy_batch(m->ctx[d], ph.first, ph.second, hf_bits, r.second - r.first,
                            theta + (size_t)r.first * ng, e_out + r.first);
  });
}

int ffq_multi_energy_units(ffq_multi_t m, int n_units, const int* problem, const uint64_t* hf_bits,
                           const int* batch, const double* const* theta, double* const* e_out, int* device_out) {
  if (!m || n_units < 0 || (n_units > 0 && (!problem || !hf_bits || !batch || !theta || !e_out)))
    return multi_fail(m, FFQ_EINVAL, "ffq_multi_energy_units: invalid argument");
  for (int u = 0; u < n_units; ++u)
    if (problem[u] < 0 || problem[u] >= (int)m->probs.size() || batch[u] < 0 || (batch[u] > 0 && (!theta[u] || !e_out[u])))
      return multi_fail(m, FFQ_EINVAL, "ffq_multi_energy_units: invalid unit " + std::to_string(u));
  // longest processing time first over the devices (shard_by_cost); ties by unit index
  const int D = (int)m->ctx.size();
  std::vector<int> ord(n_units), owner(n_units, 0);
  for (int u = 0; u < n_units; ++u) ord[u] = u;
  auto cost = [&](int u) { return m->cost[problem[u]] * batch[u]; };
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return cost(a) > cost(b); });
  std::vector<double> load(D, 0.0);
  for (int u : ord) {
    const int d = (int)(std::min_element(load.begin(), load.end()) - load.begin());
    load[d] += cost(u);
    owner[u] = d;
  }
  if (device_out)
    for (int u = 0; u < n_units; ++u) device_out[u] = owner[u];
  return on_devices(m, all_devices(m), [&](int d) {
    for (int u = 0; u < n_units; ++u) {
      if (owner[u] != d || batch[u] == 0) continue;
      const auto& ph = m->probs[problem[u]][d];
      const int rc = ffq_energy_batch(m->ctx[d], ph.first, ph.second, hf_bits[u], batch[u], theta[u], e_out[u]);
      if (rc != FFQ_OK) return rc;
    }
    return (int)FFQ_OK;
  });
}

}  // extern "C"
