// fragfield_host.cpp -- host side of the operator API (include/fragfield/*.hpp):
// Pauli algebra + Jordan-Wigner, synthetic Hamiltonians
// (BASELINE.json configs), UCCSD generators and magnitude
// ordering, the device facade over fragfield_cuda.h,
// optimizers and the FMO two-body assembly
// (reference proj/core/src/fmo.cpp:28-48).
#include <algorithm>
#include <cctype>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <limits>
#include <numeric>
#include <random>
#include <sstream>
#include <memory>
#include <string>
#include <thread>

#include "fragfield/errors.hpp"
#include "fragfield/fmo_batch.hpp"
#include "fragfield/hamiltonian.hpp"
#include "fragfield/pauli.hpp"
#include "fragfield/statevector.hpp"
#include "fragfield/uccsd.hpp"
#include "fragfield/vqe.hpp"

namespace fragfield {

namespace {
inline int popc(uint64_t v) { return __builtin_popcountll(v); }
inline Complex ipow(int k) {
  switch (k & 3) {
    case 0: return {1, 0};
    case 1: return {0, 1};
    case 2: return {-1, 0};
    default: return {0, -1};
  }
}
inline uint64_t below(int p) { return p > 0 ? ((1ULL << p) - 1ULL) : 0ULL; }

// value mapping of the pinned RNG
inline double u01(std::mt19937_64& g) { return (double)(g() >> 11) * (1.0 / 9007199254740992.0); }
inline double normal01(std::mt19937_64& g) {
  const double u1 = u01(g);
  const double u2 = u01(g);
  return std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
}
}  // namespace

// ---- Pauli algebra -------------------------------------------------------------
std::string PauliString::letters() const {
  std::string s(n_qubits, 'I');
  for (int q = 0; q < n_qubits; ++q) {
    const bool xb = (x >> q) & 1ULL, zb = (z >> q) & 1ULL;
    s[q] = xb && zb ? 'Y' : xb ? 'X' : zb ? 'Z' : 'I';
  }
  return s;
}

PauliString PauliString::parse(const std::string& letters) {
  PauliString p;
  p.n_qubits = (int)letters.size();
  if (p.n_qubits > 64) throw ContractViolation("PauliString: more than 64 qubits");
  for (int q = 0; q < p.n_qubits; ++q) {
    switch (letters[q]) {
      case 'I': break;
      case 'X': p.x |= 1ULL << q; break;
      case 'Y': p.x |= 1ULL << q; p.z |= 1ULL << q; break;
      case 'Z': p.z |= 1ULL << q; break;
      default: throw ContractViolation(std::string("PauliString: bad letter '") + letters[q] + "'");
    }
  }
  return p;
}

// P(x,z) = i^{popc(x&z)} X^x Z^z;  P1 P2 = i^{y1+y2+2 popc(z1&x2)-y3} P3
std::pair<int, PauliString> pauli_mul(const PauliString& a, const PauliString& b) {
  if (a.n_qubits != b.n_qubits) throw ContractViolation("pauli_mul: mismatched n_qubits");
  PauliString c;
  c.n_qubits = a.n_qubits;
  c.x = a.x ^ b.x;
  c.z = a.z ^ b.z;
  const int k = popc(a.x & a.z) + popc(b.x & b.z) + 2 * popc(a.z & b.x) - popc(c.x & c.z);
  return {((k % 4) + 4) % 4, c};
}

void PauliSum::add(uint64_t x, uint64_t z, Complex c) {
  if (n_ < 64 && ((x | z) >> n_)) throw ContractViolation("PauliSum: string exceeds n_qubits");
  terms_[{x, z}] += c;
}

void PauliSum::simplify(double tol) {
  for (auto it = terms_.begin(); it != terms_.end();) {
    if (std::abs(it->second) <= tol) it = terms_.erase(it);
    else ++it;
  }
}

PauliSum PauliSum::operator+(const PauliSum& o) const {
  if (o.n_ != n_) throw ContractViolation("PauliSum +: mismatched n_qubits");
  PauliSum r = *this;
  for (auto& kv : o.terms_) r.terms_[kv.first] += kv.second;
  r.simplify();
  return r;
}

PauliSum PauliSum::operator*(const PauliSum& o) const {
  if (o.n_ != n_) throw ContractViolation("PauliSum *: mismatched n_qubits");
  PauliSum r(n_);
  for (auto& a : terms_)
    for (auto& b : o.terms_) {
      auto pr = pauli_mul(PauliString{n_, a.first.first, a.first.second},
                          PauliString{n_, b.first.first, b.first.second});
      r.terms_[{pr.second.x, pr.second.z}] += a.second * b.second * ipow(pr.first);
    }
  r.simplify();
  return r;
}

PauliSum PauliSum::scaled(Complex s) const {
  PauliSum r = *this;
  for (auto& kv : r.terms_) kv.second *= s;
  return r;
}

void PauliSum::flatten(std::vector<uint64_t>& x, std::vector<uint64_t>& z, std::vector<double>& re,
                       std::vector<double>& im) const {
  for (auto& kv : terms_) {
    x.push_back(kv.first.first);
    z.push_back(kv.first.second);
    re.push_back(kv.second.real());
    im.push_back(kv.second.imag());
  }
}

std::string PauliSum::to_text() const {
  std::ostringstream os;
  os.precision(17);
  for (auto& kv : terms_)
    os << kv.second.real() << ' ' << kv.second.imag() << ' '
       << PauliString{n_, kv.first.first, kv.first.second}.letters() << '\n';
  return os.str();
}

PauliSum PauliSum::from_text(const std::string& text) {
  std::istringstream is(text);
  std::string line;
  PauliSum r(0);
  bool first = true;
  while (std::getline(is, line)) {
    if (line.empty()) continue;
    std::istringstream ls(line);
    double re, im;
    std::string letters;
    if (!(ls >> re >> im >> letters)) throw ContractViolation("PauliSum::from_text: malformed line");
    PauliString p = PauliString::parse(letters);
    if (first) { r = PauliSum(p.n_qubits); first = false; }
    if (p.n_qubits != r.n_) throw ContractViolation("PauliSum::from_text: mixed qubit counts");
    r.add(p, Complex(re, im));
  }
  r.simplify();
  return r;
}

bool PauliSum::is_hermitian(double tol) const {
  for (auto& kv : terms_)
    if (std::abs(kv.second.imag()) > tol) return false;
  return true;
}
bool PauliSum::is_antihermitian(double tol) const {
  for (auto& kv : terms_)
    if (std::abs(kv.second.real()) > tol) return false;
  return true;
}

PauliSum jordan_wigner_ladder(const LadderOp& op, int n_so) {
  if (op.index < 0 || op.index >= n_so || n_so > 64)
    throw ContractViolation("jordan_wigner: index out of range");
  PauliSum s(n_so);
  const int p = op.index;
  s.add(1ULL << p, below(p), Complex(0.5, 0.0));                              // X_p Z_<p
  s.add(1ULL << p, below(p) | (1ULL << p), Complex(0.0, op.dagger ? -0.5 : 0.5));  // Y_p Z_<p
  return s;
}

PauliSum jordan_wigner(const FermionOperator& op, int n_so) {
  PauliSum total(n_so);
  for (auto& t : op) {
    PauliSum prod(n_so);
    prod.add(0, 0, t.coef);
    for (auto& l : t.ops) prod = prod * jordan_wigner_ladder(l, n_so);
    for (auto& kv : prod.terms()) total.add(kv.first.first, kv.first.second, kv.second);
  }
  total.simplify();
  return total;
}

// ---- two-qubit reduction -----------------------------------
namespace {
// blocked index of JW qubit q (alpha first) and its inverse
int blocked_of(int q, int m) { return (q & 1) ? m + q / 2 : q / 2; }
int jw_of(int k, int m) { return k < m ? 2 * k : 2 * (k - m) + 1; }
// y = A x: y_j = parity of the modes with blocked index <= j
uint64_t parity_encode(uint64_t x, int n) {
  const int m = n / 2;
  uint64_t y = 0;
  int acc = 0;
  for (int k = 0; k < n; ++k) {
    acc ^= (int)((x >> jw_of(k, m)) & 1u);
    y |= (uint64_t)acc << k;
  }
  return y;
}
// z' = A^-T z: z'_k = z_(jw of k) xor z_(jw of k+1)
uint64_t parity_encode_z(uint64_t z, int n) {
  const int m = n / 2;
  uint64_t out = 0;
  for (int k = 0; k < n; ++k) {
    int v = (int)((z >> jw_of(k, m)) & 1u);
    if (k + 1 < n) v ^= (int)((z >> jw_of(k + 1, m)) & 1u);
    out |= (uint64_t)v << k;
  }
  return out;
}
// drop bits t1 < t2 of v
uint64_t drop_two(uint64_t v, int t1, int t2) {
  const uint64_t lo = v & ((1ULL << t1) - 1);
  const uint64_t mid = (v >> (t1 + 1)) & ((1ULL << (t2 - t1 - 1)) - 1);
  const uint64_t hi = t2 + 1 < 64 ? v >> (t2 + 1) : 0;
  return lo | (mid << t1) | (hi << (t2 - 1));
}
}  // namespace

PauliSum reduce_two_qubits(const PauliSum& op, int n_so, int n_alpha, int n_beta) {
  if (n_so < 4 || n_so % 2 || n_so > 64 || op.n_qubits() != n_so)
    throw ContractViolation("reduce_two_qubits: need an even n_so in [4, 64] matching the operator");
  if (n_alpha < 0 || n_beta < 0 || n_alpha > n_so / 2 || n_beta > n_so / 2)
    throw ContractViolation("reduce_two_qubits: electron counts out of range");
  const int m = n_so / 2, t1 = m - 1, t2 = n_so - 1;
  const int y1 = n_alpha & 1, y2 = (n_alpha + n_beta) & 1;  // parity-qubit eigenvalues (-1)^y
  (void)blocked_of;
  PauliSum out(n_so - 2);
  for (const auto& kv : op.terms()) {
    const uint64_t a = kv.first.first, b = kv.first.second;
    const uint64_t a2 = parity_encode(a, n_so), b2 = parity_encode_z(b, n_so);
    if (((a2 >> t1) & 1u) || ((a2 >> t2) & 1u))
      throw ContractViolation("reduce_two_qubits: a term flips a conserved parity qubit (operator does not "
                              "commute with the N_alpha / N parities)");
    // c i^{|a&b|} X^a Z^b -> c i^{|a&b|} X^a2 Z^b2 = c i^{|a&b| - |a2&b2|} P(a2, b2)
    const int k = (__builtin_popcountll(a & b) - __builtin_popcountll(a2 & b2)) & 3;
    Complex c = kv.second;
    static const Complex ik[4] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
    c *= ik[k];
    if ((((b2 >> t1) & 1u) && y1) ^ (((b2 >> t2) & 1u) && y2)) c = -c;  // Z on a parity qubit -> eigenvalue
    out.add(drop_two(a2, t1, t2), drop_two(b2, t1, t2), c);
  }
  out.simplify();
  return out;
}

uint64_t reduce_two_qubits_basis(uint64_t jw_bits, int n_so) {
  if (n_so < 4 || n_so % 2 || n_so > 64) throw ContractViolation("reduce_two_qubits_basis: need an even n_so in [4, 64]");
  return drop_two(parity_encode(jw_bits, n_so), n_so / 2 - 1, n_so - 1);
}

// ---- Hamiltonians --------------------------------------------------------------
SpatialIntegrals synthetic_integrals(int m, uint64_t seed, double sigma_h, double sigma_g) {
  if (m < 1 || m > 32) throw ContractViolation("synthetic_integrals: m out of range");
  SpatialIntegrals I;
  I.m = m;
  I.h.assign((size_t)m * m, 0.0);
  I.g.assign((size_t)m * m * m * m, 0.0);
  std::mt19937_64 gen(seed);
  for (int p = 0; p < m; ++p)
    for (int q = 0; q <= p; ++q) {
      const double v = sigma_h * normal01(gen);
      I.h[(size_t)p * m + q] = v;
      I.h[(size_t)q * m + p] = v;
    }
  auto G = [&](int a, int b, int c, int d) -> double& {
    return I.g[(((size_t)a * m + b) * m + c) * m + d];
  };
  for (int p = 0; p < m; ++p)
    for (int q = 0; q <= p; ++q)
      for (int r = 0; r <= p; ++r) {
        const int smax = (r == p) ? q : r;
        for (int s = 0; s <= smax; ++s) {
          const double v = sigma_g * normal01(gen);
          G(p, q, r, s) = v; G(q, p, r, s) = v; G(p, q, s, r) = v; G(q, p, s, r) = v;
          G(r, s, p, q) = v; G(s, r, p, q) = v; G(r, s, q, p) = v; G(s, r, q, p) = v;
        }
      }
  return I;
}

void write_fcidump(const std::string& path, const SpatialIntegrals& I, int n_elec, int ms2) {
  const int m = I.m;
  if (m < 1 || I.h.size() != (size_t)m * m || I.g.size() != (size_t)m * m * m * m)
    throw ContractViolation("write_fcidump: integral shapes");
  std::FILE* f = std::fopen(path.c_str(), "w");
  if (!f) throw std::runtime_error("write_fcidump: cannot open " + path);
  std::fprintf(f, " &FCI NORB=%d,NELEC=%d,MS2=%d,\n  ORBSYM=", m, n_elec, ms2);
  for (int i = 0; i < m; ++i) std::fprintf(f, "1,");
  std::fprintf(f, "\n  ISYM=1,\n &END\n");
  auto G = [&](int a, int b, int c, int d) { return I.g[(((size_t)a * m + b) * m + c) * m + d]; };
  for (int i = 0; i < m; ++i)
    for (int j = 0; j <= i; ++j)
      for (int k = 0; k < m; ++k)
        for (int l = 0; l <= k; ++l) {
          if (i * (i + 1) / 2 + j < k * (k + 1) / 2 + l) continue;  // ij >= kl
          const double v = G(i, j, k, l);
          if (v != 0.0) std::fprintf(f, "%.17g %d %d %d %d\n", v, i + 1, j + 1, k + 1, l + 1);
        }
  for (int i = 0; i < m; ++i)
    for (int j = 0; j <= i; ++j)
      if (I.h[(size_t)i * m + j] != 0.0) std::fprintf(f, "%.17g %d %d 0 0\n", I.h[(size_t)i * m + j], i + 1, j + 1);
  std::fprintf(f, "%.17g 0 0 0 0\n", I.e_const);
  std::fclose(f);
}

Fcidump read_fcidump(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("read_fcidump: cannot open " + path);
  std::string line, header;
  int ln = 0;
  bool done = false;
  while (!done && std::getline(in, line)) {
    ++ln;
    header += line + " ";
    std::string up = line;
    for (auto& ch : up) ch = (char)std::toupper((unsigned char)ch);
    if (up.find("&END") != std::string::npos || up.find("/") != std::string::npos) done = true;
  }
  if (!done) throw ParseError("read_fcidump: header without &END", ln);
  auto key = [&](const char* k, int dflt, bool required) {
    std::string up = header;
    for (auto& ch : up) ch = (char)std::toupper((unsigned char)ch);
    const size_t p = up.find(k);
    if (p == std::string::npos) {
      if (required) throw ParseError(std::string("read_fcidump: header lacks ") + k, ln);
      return dflt;
    }
    size_t q = up.find('=', p);
    if (q == std::string::npos) throw ParseError(std::string("read_fcidump: malformed ") + k, ln);
    return std::atoi(header.c_str() + q + 1);
  };
  Fcidump F;
  const int m = key("NORB", 0, true);
  F.n_elec = key("NELEC", 0, true);
  F.ms2 = key("MS2", 0, false);
  if (m < 1 || m > 64) throw ParseError("read_fcidump: NORB out of range", ln);
  F.ints.m = m;
  F.ints.h.assign((size_t)m * m, 0.0);
  F.ints.g.assign((size_t)m * m * m * m, 0.0);
  auto G = [&](int a, int b, int c, int d) -> double& { return F.ints.g[(((size_t)a * m + b) * m + c) * m + d]; };
  while (std::getline(in, line)) {
    ++ln;
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    std::istringstream ss(line);
    double v;
    int i, j, k, l;
    if (!(ss >> v >> i >> j >> k >> l)) throw ParseError("read_fcidump: malformed integral line", ln);
    if (i < 0 || j < 0 || k < 0 || l < 0 || i > m || j > m || k > m || l > m)
      throw ParseError("read_fcidump: orbital index out of range", ln);
    if (i == 0 && j == 0 && k == 0 && l == 0) {
      F.ints.e_const = v;
    } else if (k == 0 && l == 0) {
      if (i == 0 || j == 0) throw ParseError("read_fcidump: malformed one-electron line", ln);
      F.ints.h[(size_t)(i - 1) * m + (j - 1)] = v;
      F.ints.h[(size_t)(j - 1) * m + (i - 1)] = v;
    } else {
      if (i == 0 || j == 0 || k == 0 || l == 0) throw ParseError("read_fcidump: malformed two-electron line", ln);
      const int a = i - 1, b = j - 1, c = k - 1, d = l - 1;
      G(a, b, c, d) = v; G(b, a, c, d) = v; G(a, b, d, c) = v; G(b, a, d, c) = v;
      G(c, d, a, b) = v; G(d, c, a, b) = v; G(c, d, b, a) = v; G(d, c, b, a) = v;
    }
  }
  return F;
}

void write_state_dump(const std::string& path, int n_qubits, const std::vector<std::complex<double>>& amps) {
  if (n_qubits < 0 || n_qubits > 40 || amps.size() != (size_t)1 << n_qubits)
    throw ContractViolation("write_state_dump: need 2^n_qubits amplitudes");
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("write_state_dump: cannot open " + path);
  const int64_t n = n_qubits;  // x86-64 and aarch64 hosts are little-endian
  out.write(reinterpret_cast<const char*>(&n), sizeof(n));
  out.write(reinterpret_cast<const char*>(amps.data()), (std::streamsize)(amps.size() * sizeof(amps[0])));
  if (!out) throw std::runtime_error("write_state_dump: write failed");
}

std::vector<std::complex<double>> read_state_dump(const std::string& path, int* n_qubits) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("read_state_dump: cannot open " + path);
  int64_t n = -1;
  in.read(reinterpret_cast<char*>(&n), sizeof(n));
  if (!in || n < 0 || n > 40) throw ParseError("read_state_dump: bad header", 0);
  std::vector<std::complex<double>> a((size_t)1 << n);
  in.read(reinterpret_cast<char*>(a.data()), (std::streamsize)(a.size() * sizeof(a[0])));
  if (!in) throw ParseError("read_state_dump: truncated amplitude array", 0);
  if (in.peek() != std::char_traits<char>::eof()) throw ParseError("read_state_dump: trailing bytes", 0);
  if (n_qubits) *n_qubits = (int)n;
  return a;
}

std::vector<double> uniform_vector(uint64_t seed, int count, double lo, double hi) {
  std::mt19937_64 gen(seed);
  std::vector<double> v((size_t)std::max(0, count));
  for (auto& e : v) e = lo + (hi - lo) * u01(gen);
  return v;
}

SpatialIntegrals ao_to_mo(const SpatialIntegrals& ao, const std::vector<double>& C, int m,
                          const std::vector<double>& v_esp) {
  const int n = ao.m;
  const size_t N = (size_t)n;
  if (n < 1 || m < 1 || m > n) throw ContractViolation("ao_to_mo: need 1 <= m <= n AO functions");
  if (ao.h.size() != N * N || ao.g.size() != N * N * N * N || C.size() != N * (size_t)m)
    throw ContractViolation("ao_to_mo: integral or coefficient shapes");
  if (!v_esp.empty() && v_esp.size() != N * N) throw ContractViolation("ao_to_mo: v_esp shape");
  const size_t M = (size_t)m;
  SpatialIntegrals mo;
  mo.m = m;
  mo.e_const = ao.e_const;
  // one-electron: C^T (h + V) C
  std::vector<double> hv(ao.h);
  if (!v_esp.empty())
    for (size_t k = 0; k < N * N; ++k) hv[k] += v_esp[k];
  std::vector<double> t1(N * M, 0.0);
  for (size_t a = 0; a < N; ++a)
    for (size_t b = 0; b < N; ++b)
      for (size_t q = 0; q < M; ++q) t1[a * M + q] += hv[a * N + b] * C[b * M + q];
  mo.h.assign(M * M, 0.0);
  for (size_t p = 0; p < M; ++p)
    for (size_t a = 0; a < N; ++a)
      for (size_t q = 0; q < M; ++q) mo.h[p * M + q] += C[a * M + p] * t1[a * M + q];
  // two-electron: four quarter transformations, one index at a time
  // g1[a][b][c][s] = sum_d g[a][b][c][d] C[d][s], then c -> r, b -> q, a -> p
  std::vector<double> g1(N * N * N * M, 0.0);
  for (size_t abc = 0; abc < N * N * N; ++abc)
    for (size_t d = 0; d < N; ++d) {
      const double v = ao.g[abc * N + d];
      if (v == 0.0) continue;
      for (size_t s2 = 0; s2 < M; ++s2) g1[abc * M + s2] += v * C[d * M + s2];
    }
  std::vector<double> g2(N * N * M * M, 0.0);  // [a][b][r][s]
  for (size_t ab = 0; ab < N * N; ++ab)
    for (size_t c = 0; c < N; ++c)
      for (size_t r = 0; r < M; ++r) {
        const double cr = C[c * M + r];
        if (cr == 0.0) continue;
        for (size_t s2 = 0; s2 < M; ++s2) g2[(ab * M + r) * M + s2] += cr * g1[(ab * N + c) * M + s2];
      }
  std::vector<double> g3(N * M * M * M, 0.0);  // [a][q][r][s]
  for (size_t a = 0; a < N; ++a)
    for (size_t b = 0; b < N; ++b)
      for (size_t q = 0; q < M; ++q) {
        const double bq = C[b * M + q];
        if (bq == 0.0) continue;
        for (size_t rs = 0; rs < M * M; ++rs) g3[(a * M + q) * M * M + rs] += bq * g2[(a * N + b) * M * M + rs];
      }
  mo.g.assign(M * M * M * M, 0.0);
  for (size_t a = 0; a < N; ++a)
    for (size_t p = 0; p < M; ++p) {
      const double ap = C[a * M + p];
      if (ap == 0.0) continue;
      for (size_t qrs = 0; qrs < M * M * M; ++qrs) mo.g[p * M * M * M + qrs] += ap * g3[a * M * M * M + qrs];
    }
  return mo;
}

FrozenCore freeze_core(const SpatialIntegrals& mo, int n_frozen, int n_elec) {
  const int m = mo.m;
  if (n_frozen < 0 || 2 * n_frozen > n_elec || n_frozen > m)
    throw ContractViolation("freeze_core: n_frozen exceeds the occupied orbitals");
  const size_t M = (size_t)m;
  auto G = [&](int p, int q, int r, int s2) { return mo.g[((p * M + q) * M + r) * M + s2]; };
  FrozenCore F;
  double ef = 0.0;
  for (int c = 0; c < n_frozen; ++c) {
    ef += 2.0 * mo.h[c * M + c];
    for (int d = 0; d < n_frozen; ++d) ef += 2.0 * G(c, c, d, d) - G(c, d, d, c);
  }
  const int ma = m - n_frozen;
  const size_t A = (size_t)ma;
  F.active.m = ma;
  F.active.h.assign(A * A, 0.0);
  F.active.g.assign(A * A * A * A, 0.0);
  for (int p = 0; p < ma; ++p)
    for (int q = 0; q < ma; ++q) {
      double v = mo.h[(p + n_frozen) * M + (q + n_frozen)];
      for (int c = 0; c < n_frozen; ++c)
        v += 2.0 * G(p + n_frozen, q + n_frozen, c, c) - G(p + n_frozen, c, c, q + n_frozen);
      F.active.h[p * A + q] = v;
    }
  for (int p = 0; p < ma; ++p)
    for (int q = 0; q < ma; ++q)
      for (int r = 0; r < ma; ++r)
        for (int s2 = 0; s2 < ma; ++s2)
          F.active.g[((p * A + q) * A + r) * A + s2] = G(p + n_frozen, q + n_frozen, r + n_frozen, s2 + n_frozen);
  F.e_frozen = ef;
  F.active.e_const = mo.e_const + ef;
  F.n_elec_active = n_elec - 2 * n_frozen;
  return F;
}

SpinOrbitalHamiltonian to_spin_orbitals(const SpatialIntegrals& I, int n_elec) {
  const int m = I.m, n = 2 * m;
  if (n_elec < 0 || n_elec > n) throw ContractViolation("to_spin_orbitals: bad electron count");
  SpinOrbitalHamiltonian H;
  H.n_so = n;
  H.n_elec = n_elec;
  H.e_const = I.e_const;
  H.h.assign((size_t)n * n, 0.0);
  H.g.assign((size_t)n * n * n * n, 0.0);
  for (int p = 0; p < n; ++p)
    for (int q = 0; q < n; ++q)
      if ((p & 1) == (q & 1)) H.h[(size_t)p * n + q] = I.h[(size_t)(p >> 1) * m + (q >> 1)];
  for (int p = 0; p < n; ++p)
    for (int q = 0; q < n; ++q)
      for (int r = 0; r < n; ++r)
        for (int s = 0; s < n; ++s)
          if ((p & 1) == (r & 1) && (q & 1) == (s & 1))
            H.g[(((size_t)p * n + q) * n + r) * n + s] =
                I.g[(((size_t)(p >> 1) * m + (r >> 1)) * m + (q >> 1)) * m + (s >> 1)];
  return H;
}

PauliSum qubit_hamiltonian(const SpinOrbitalHamiltonian& H) {
  const int n = H.n_so;
  if (n > 64) throw ContractViolation("qubit_hamiltonian: more than 64 spin orbitals");
  std::vector<PauliSum> a, ad;
  for (int p = 0; p < n; ++p) {
    a.push_back(jordan_wigner_ladder({p, false}, n));
    ad.push_back(jordan_wigner_ladder({p, true}, n));
  }
  PauliSum out(n);
  if (H.e_const != 0.0) out.add(0, 0, H.e_const);
  auto accumulate = [&](const PauliSum& s) {
    for (auto& kv : s.terms()) out.add(kv.first.first, kv.first.second, kv.second);
  };
  for (int p = 0; p < n; ++p)
    for (int q = 0; q < n; ++q) {
      const double v = H.h[(size_t)p * n + q];
      if (v != 0.0) accumulate((ad[p] * a[q]).scaled(v));
    }
  std::vector<PauliSum> asr((size_t)n * n, PauliSum(n));  // a_s a_r
  for (int s = 0; s < n; ++s)
    for (int r = 0; r < n; ++r)
      if (r != s) asr[(size_t)s * n + r] = a[s] * a[r];
  for (int p = 0; p < n; ++p)
    for (int q = 0; q < n; ++q) {
      if (p == q) continue;
      const PauliSum apq = ad[p] * ad[q];
      for (int r = 0; r < n; ++r)
        for (int s = 0; s < n; ++s) {
          if (r == s) continue;
          const double v = H.g[(((size_t)p * n + q) * n + r) * n + s];
          if (v == 0.0) continue;
          accumulate((apq * asr[(size_t)s * n + r]).scaled(0.5 * v));
        }
    }
  out.simplify();
  return out;
}

PauliSum random_pauli_hamiltonian(int n_qubits, int n_terms, uint64_t seed, double sigma) {
  if (n_qubits < 1 || n_qubits > 64) throw ContractViolation("random_pauli_hamiltonian: bad n");
  std::mt19937_64 gen(seed);
  PauliSum H(n_qubits);
  for (int t = 0; t < n_terms; ++t) {
    uint64_t x = 0, z = 0;
    for (int q = 0; q < n_qubits; ++q) {
      const uint64_t l = gen() >> 62;  // 0 I, 1 X, 2 Y, 3 Z
      if (l == 1 || l == 2) x |= 1ULL << q;
      if (l == 2 || l == 3) z |= 1ULL << q;
    }
    H.add(x, z, sigma * normal01(gen));
  }
  H.simplify();
  return H;
}

// ---- UCCSD ---------------------------------------------------------------------
std::vector<Generator> build_generators(int n_so, int n_elec) {
  if (n_elec < 0 || n_elec > n_so || n_so > 64) throw ContractViolation("build_generators: bad sizes");
  std::vector<Excitation> ex;
  for (int i = 0; i < n_elec; ++i)
    for (int a = n_elec; a < n_so; ++a)
      if ((i & 1) == (a & 1)) ex.push_back({1, i, -1, a, -1});
  for (int i = 0; i < n_elec; ++i)
    for (int j = i + 1; j < n_elec; ++j)
      for (int a = n_elec; a < n_so; ++a)
        for (int b = a + 1; b < n_so; ++b)
          if ((i & 1) + (j & 1) == (a & 1) + (b & 1)) ex.push_back({2, i, j, a, b});
  std::vector<Generator> gens;
  gens.reserve(ex.size());
  for (size_t k = 0; k < ex.size(); ++k) {
    const Excitation& e = ex[k];
    FermionOperator op;
    if (e.kind == 1) {
      op.push_back({Complex(1, 0), {{e.a, true}, {e.i, false}}});
      op.push_back({Complex(-1, 0), {{e.i, true}, {e.a, false}}});
    } else {
      op.push_back({Complex(1, 0), {{e.a, true}, {e.b, true}, {e.j, false}, {e.i, false}}});
      op.push_back({Complex(-1, 0), {{e.i, true}, {e.j, true}, {e.b, false}, {e.a, false}}});
    }
    gens.push_back({(int)k, e, jordan_wigner(op, n_so)});
  }
  return gens;
}

TrotterPlan magnitude_order(const std::vector<Generator>& gens, const std::vector<double>& amps,
                            int n_qubits) {
  if (amps.size() > gens.size()) throw ContractViolation("magnitude_order: more amplitudes than generators");
  TrotterPlan P;
  P.n_qubits = n_qubits;
  P.generators = gens;
  P.order.resize(gens.size());
  std::iota(P.order.begin(), P.order.end(), 0);
  auto amp = [&](int g) { return g < (int)amps.size() ? std::abs(amps[g]) : 0.0; };
  std::stable_sort(P.order.begin(), P.order.end(), [&](int u, int v) {
    const double fu = amp(u), fv = amp(v);
    if (fu != fv) return fu > fv;
    return u < v;
  });
  return P;
}

std::vector<double> TrotterPlan::plan_theta(const std::vector<double>& amps) const {
  if (amps.size() != generators.size()) throw ContractViolation("plan_theta: amplitude count mismatch");
  std::vector<double> t(order.size());
  for (size_t s = 0; s < order.size(); ++s) t[s] = amps[order[s]];
  return t;
}

void TrotterPlan::flatten(std::vector<int64_t>& off, std::vector<uint64_t>& x,
                          std::vector<uint64_t>& z, std::vector<double>& re,
                          std::vector<double>& im) const {
  off.assign(1, 0);
  for (int gid : order) {
    generators[gid].image.flatten(x, z, re, im);
    off.push_back((int64_t)x.size());
  }
}

uint64_t hf_bits(int n_elec) {
  if (n_elec < 0 || n_elec > 63) throw ContractViolation("hf_bits: electron count out of range");
  return (n_elec == 0) ? 0ULL : ((1ULL << n_elec) - 1ULL);
}

// ---- device facade ---------------------------------------------------------------
void check_ffq(int rc, ffq_ctx_t ctx) {
  if (rc == FFQ_OK) return;
  const std::string msg = ffq_last_error(ctx);
  if (rc == FFQ_EINVAL || rc == FFQ_ENONHERMITIAN) throw ContractViolation(msg);
  throw DeviceError(msg, rc);
}

Device::Device(int ordinal) : ordinal_(ordinal) { check_ffq(ffq_ctx_create(ordinal, &ctx_), nullptr); }
Device::~Device() { ffq_ctx_destroy(ctx_); }
void Device::synchronize() const { check_ffq(ffq_ctx_synchronize(ctx_), ctx_); }
int Device::count() {
  int n = 0;
  return ffq_device_count(&n) == FFQ_OK ? n : 0;
}

DeviceHamiltonian::DeviceHamiltonian(Device& dev, const PauliSum& H) : dev_(dev), n_(H.n_qubits()) {
  std::vector<uint64_t> x, z;
  std::vector<double> re, im;
  H.flatten(x, z, re, im);
  check_ffq(ffq_ham_upload(dev.handle(), n_, (int64_t)x.size(), x.data(), z.data(), re.data(),
                           im.data(), &h_),
            dev.handle());
}
DeviceHamiltonian::~DeviceHamiltonian() { ffq_ham_destroy(h_); }
int DeviceHamiltonian::n_groups() const {
  int g = 0;
  ffq_ham_info(h_, &g, nullptr, nullptr);
  return g;
}
int64_t DeviceHamiltonian::n_classes() const {
  int64_t c = 0;
  ffq_ham_info(h_, nullptr, nullptr, &c);
  return c;
}

DevicePlan::DevicePlan(Device& dev, const TrotterPlan& plan) : dev_(dev), plan_(plan) {
  std::vector<int64_t> off;
  std::vector<uint64_t> x, z;
  std::vector<double> re, im;
  plan.flatten(off, x, z, re, im);
  check_ffq(ffq_plan_upload(dev.handle(), plan.n_qubits, (int)plan.order.size(), off.data(),
                            x.data(), z.data(), re.data(), im.data(), &p_),
            dev.handle());
}
DevicePlan::~DevicePlan() { ffq_plan_destroy(p_); }
int DevicePlan::n_fused() const {
  int f = 0;
  ffq_plan_info(p_, &f, nullptr);
  return f;
}
int DevicePlan::n_string_ops() const {
  int s = 0;
  ffq_plan_info(p_, nullptr, &s);
  return s;
}

Statevector::Statevector(Device& dev, int n_qubits, int batch) : dev_(dev), n_(n_qubits), batch_(batch) {
  check_ffq(ffq_state_alloc(dev.handle(), n_qubits, batch, &s_), dev.handle());
}
Statevector::~Statevector() { ffq_state_free(s_); }
void Statevector::set_basis(uint64_t bits) { check_ffq(ffq_state_set_basis(s_, bits), dev_.handle()); }
void Statevector::apply_pauli_rotation(const PauliString& p, double theta) {
  if (p.n_qubits != n_) throw ContractViolation("apply_pauli_rotation: qubit count mismatch");
  check_ffq(ffq_state_apply_pauli_rotation(s_, p.x, p.z, theta), dev_.handle());
}
void Statevector::apply_pauli_rotations(const std::vector<PauliString>& ps, const std::vector<double>& theta) {
  if (ps.size() != theta.size()) throw ContractViolation("apply_pauli_rotations: one angle per string");
  std::vector<uint64_t> x(ps.size()), z(ps.size());
  for (size_t r = 0; r < ps.size(); ++r) {
    if (ps[r].n_qubits != n_) throw ContractViolation("apply_pauli_rotations: qubit count mismatch");
    x[r] = ps[r].x;
    z[r] = ps[r].z;
  }
  check_ffq(ffq_state_apply_pauli_rotations(s_, (int)ps.size(), x.data(), z.data(), theta.data()), dev_.handle());
}
void Statevector::apply_plan(const DevicePlan& plan, const std::vector<double>& theta) {
  if (theta.size() != plan.plan().order.size() * (size_t)batch_)
    throw ContractViolation("apply_plan: theta must be [batch][n_gen]");
  check_ffq(ffq_state_apply_plan(s_, plan.handle(), theta.data()), dev_.handle());
}
std::vector<double> Statevector::expectation(const DeviceHamiltonian& H) const {
  std::vector<double> re(batch_), im(batch_);
  check_ffq(ffq_state_expectation(s_, H.handle(), re.data(), im.data()), dev_.handle());
  for (double v : im)
    if (std::abs(v) > 1e-10) throw ContractViolation("expectation: imaginary residue above 1e-10");
  return re;
}
std::vector<Complex> Statevector::download() const {
  std::vector<Complex> v((size_t)batch_ << n_);
  check_ffq(ffq_state_download(s_, reinterpret_cast<double*>(v.data())), dev_.handle());
  return v;
}
void Statevector::upload(const std::vector<Complex>& amps) {
  if (amps.size() != ((size_t)batch_ << n_)) throw ContractViolation("upload: size mismatch");
  check_ffq(ffq_state_upload(s_, reinterpret_cast<const double*>(amps.data())), dev_.handle());
}

std::vector<double> energy_batch(Device& dev, const DevicePlan& plan, const DeviceHamiltonian& H,
                                 uint64_t hf, const std::vector<double>& theta, int batch) {
  const size_t ng = plan.plan().order.size();
  if (theta.size() != ng * (size_t)batch) throw ContractViolation("energy_batch: theta must be [batch][n_gen]");
  std::vector<double> e((size_t)batch);
  check_ffq(ffq_energy_batch(dev.handle(), plan.handle(), H.handle(), hf, batch, theta.data(), e.data()),
            dev.handle());
  return e;
}

void prepare(Device& dev, const DevicePlan& plan, const DeviceHamiltonian& H, uint64_t hf) {
  check_ffq(ffq_energy_prepare(dev.handle(), plan.handle(), H.handle(), hf), dev.handle());
}

double energy_trotter(Device& dev, const std::vector<double>& amps, const DevicePlan& plan,
                      const DeviceHamiltonian& H, uint64_t hf) {
  return energy_batch(dev, plan, H, hf, plan.plan().plan_theta(amps), 1)[0];
}

double energy_exact(Device& dev, const std::vector<double>& amps, const DevicePlan& plan,
                    const DeviceHamiltonian& H, uint64_t hf, double tol) {
  const std::vector<double> th = plan.plan().plan_theta(amps);
  double e = 0.0;
  check_ffq(ffq_energy_exact(dev.handle(), plan.handle(), H.handle(), hf, th.data(), tol, &e), dev.handle());
  return e;
}

GroundState lanczos_ground(Device& dev, const DeviceHamiltonian& H, uint64_t hf, double tol, int max_iter) {
  GroundState g;
  check_ffq(ffq_lanczos_ground(dev.handle(), H.handle(), hf, tol, max_iter, &g.energy, &g.iterations,
                               &g.dimension),
            dev.handle());
  return g;
}

// ---- optimizers ------------------------------------------------------------------
namespace {

struct Counted {
  const Objective& f;
  int evals = 0;
  int max_evals;
  double best = std::numeric_limits<double>::infinity();
  std::vector<double> best_x;
  double operator()(const std::vector<double>& x) {
    ++evals;
    const double v = f(x);
    if (v < best) { best = v; best_x = x; }
    return v;
  }
  bool exhausted() const { return evals >= max_evals; }
};

// Brent's method on f(x0 + t d) after a golden-section bracket.
double line_minimize(Counted& F, std::vector<double>& x, const std::vector<double>& d, double fx,
                     double step) {
  const double gold = 1.618033988749895, cgold = 0.3819660112501051, tiny = 1e-20;
  auto at = [&](double t) {
    std::vector<double> y(x);
    for (size_t i = 0; i < y.size(); ++i) y[i] += t * d[i];
    return F(y);
  };
  double a = 0.0, b = step, fa = fx, fb = at(b);
  if (fb > fa) { std::swap(a, b); std::swap(fa, fb); }
  double c = b + gold * (b - a), fc = at(c);
  while (fb > fc && !F.exhausted()) {
    const double r = (b - a) * (fb - fc), q = (b - c) * (fb - fa);
    double u = b - ((b - c) * q - (b - a) * r) / (2.0 * std::copysign(std::max(std::abs(q - r), tiny), q - r));
    const double ulim = b + 100.0 * (c - b);
    double fu;
    if ((b - u) * (u - c) > 0.0) {
      fu = at(u);
      if (fu < fc) { a = b; fa = fb; b = u; fb = fu; break; }
      if (fu > fb) { c = u; fc = fu; break; }
      u = c + gold * (c - b); fu = at(u);
    } else if ((c - u) * (u - ulim) > 0.0) {
      fu = at(u);
      if (fu < fc) { b = c; c = u; u = c + gold * (c - b); fb = fc; fc = fu; fu = at(u); }
    } else if ((u - ulim) * (ulim - c) >= 0.0) {
      u = ulim; fu = at(u);
    } else {
      u = c + gold * (c - b); fu = at(u);
    }
    a = b; b = c; c = u; fa = fb; fb = fc; fc = fu;
  }
  // Brent
  double lo = std::min(a, c), hi = std::max(a, c);
  double xb = b, w = b, v = b, fxb = fb, fw = fb, fv = fb, e = 0.0, dd = 0.0;
  for (int it = 0; it < 100 && !F.exhausted(); ++it) {
    const double xm = 0.5 * (lo + hi);
    const double tol1 = 1e-8 * std::abs(xb) + 1e-12, tol2 = 2.0 * tol1;
    if (std::abs(xb - xm) <= tol2 - 0.5 * (hi - lo)) break;
    if (std::abs(e) > tol1) {
      double r = (xb - w) * (fxb - fv), q = (xb - v) * (fxb - fw), p = (xb - v) * q - (xb - w) * r;
      q = 2.0 * (q - r);
      if (q > 0.0) p = -p;
      q = std::abs(q);
      const double etemp = e;
      e = dd;
      if (std::abs(p) >= std::abs(0.5 * q * etemp) || p <= q * (lo - xb) || p >= q * (hi - xb)) {
        e = (xb >= xm) ? lo - xb : hi - xb;
        dd = cgold * e;
      } else {
        dd = p / q;
        const double u = xb + dd;
        if (u - lo < tol2 || hi - u < tol2) dd = std::copysign(tol1, xm - xb);
      }
    } else {
      e = (xb >= xm) ? lo - xb : hi - xb;
      dd = cgold * e;
    }
    const double u = std::abs(dd) >= tol1 ? xb + dd : xb + std::copysign(tol1, dd);
    const double fu = at(u);
    if (fu <= fxb) {
      if (u >= xb) lo = xb; else hi = xb;
      v = w; w = xb; xb = u; fv = fw; fw = fxb; fxb = fu;
    } else {
      if (u < xb) lo = u; else hi = u;
      if (fu <= fw || w == xb) { v = w; w = u; fv = fw; fw = fu; }
      else if (fu <= fv || v == xb || v == w) { v = u; fv = fu; }
    }
  }
  if (fxb < fx) {
    for (size_t i = 0; i < x.size(); ++i) x[i] += xb * d[i];
    return fxb;
  }
  return fx;
}

}  // namespace

OptimizeResult powell_minimize(const Objective& f, std::vector<double> x, const OptimizerOptions& opts) {
  const size_t n = x.size();
  Counted F{f, 0, opts.max_evals};
  OptimizeResult R;
  std::vector<std::vector<double>> dirs(n, std::vector<double>(n, 0.0));
  for (size_t i = 0; i < n; ++i) dirs[i][i] = 1.0;
  double fx = F(x);
  while (!F.exhausted()) {
    ++R.n_iterations;
    const double f0 = fx;
    const std::vector<double> x0 = x;
    size_t ibig = 0;
    double big = 0.0;
    for (size_t i = 0; i < n && !F.exhausted(); ++i) {
      const double fold = fx;
      fx = line_minimize(F, x, dirs[i], fx, opts.initial_step);
      if (fold - fx > big) { big = fold - fx; ibig = i; }
    }
    if (f0 - fx <= opts.ftol) { R.converged = true; break; }
    std::vector<double> dnew(n), xe(n);
    for (size_t i = 0; i < n; ++i) { dnew[i] = x[i] - x0[i]; xe[i] = 2.0 * x[i] - x0[i]; }
    const double fe = F(xe);
    if (fe < f0) {
      const double t = 2.0 * (f0 - 2.0 * fx + fe) * (f0 - fx - big) * (f0 - fx - big) -
                       big * (f0 - fe) * (f0 - fe);
      if (t < 0.0) {
        fx = line_minimize(F, x, dnew, fx, 1.0);
        dirs[ibig] = dirs[n - 1];
        dirs[n - 1] = dnew;
      }
    }
  }
  R.energy = F.best;
  R.x = F.best_x;
  R.n_evals = F.evals;
  return R;
}

OptimizeResult neldermead_minimize(const Objective& f, std::vector<double> x0,
                                   const OptimizerOptions& opts) {
  const size_t n = x0.size();
  Counted F{f, 0, opts.max_evals};
  OptimizeResult R;
  // adaptive coefficients (Gao & Han)
  const double dn = (double)std::max<size_t>(n, 1);
  const double alpha = 1.0, beta = 1.0 + 2.0 / dn, gamma = 0.75 - 0.5 / dn, delta = 1.0 - 1.0 / dn;
  std::vector<std::vector<double>> s(n + 1, x0);
  std::vector<double> fs(n + 1);
  for (size_t i = 0; i < n; ++i) s[i + 1][i] += opts.initial_step;
  for (size_t i = 0; i <= n; ++i) fs[i] = F(s[i]);
  std::vector<size_t> idx(n + 1);
  while (!F.exhausted()) {
    ++R.n_iterations;
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return fs[a] < fs[b]; });
    const size_t ib = idx[0], iw = idx[n], isw = idx[n > 0 ? n - 1 : 0];
    double xspread = 0.0;
    for (size_t i = 0; i <= n; ++i)
      for (size_t k = 0; k < n; ++k) xspread = std::max(xspread, std::abs(s[i][k] - s[ib][k]));
    if (fs[iw] - fs[ib] <= opts.ftol && xspread <= std::max(opts.xtol, 1e-4)) { R.converged = true; break; }
    std::vector<double> c(n, 0.0);
    for (size_t i = 0; i <= n; ++i)
      if (i != iw)
        for (size_t k = 0; k < n; ++k) c[k] += s[i][k] / dn;
    auto lerp = [&](double t) {
      std::vector<double> y(n);
      for (size_t k = 0; k < n; ++k) y[k] = c[k] + t * (s[iw][k] - c[k]);
      return y;
    };
    std::vector<double> xr = lerp(-alpha);
    const double fr = F(xr);
    if (fr < fs[ib]) {
      std::vector<double> xe = lerp(-alpha * beta);
      const double fe = F(xe);
      if (fe < fr) { s[iw] = xe; fs[iw] = fe; } else { s[iw] = xr; fs[iw] = fr; }
    } else if (fr < fs[isw]) {
      s[iw] = xr; fs[iw] = fr;
    } else {
      const bool outside = fr < fs[iw];
      std::vector<double> xc = lerp(outside ? -alpha * gamma : gamma);
      const double fc = F(xc);
      if (fc < std::min(fr, fs[iw])) {
        s[iw] = xc; fs[iw] = fc;
      } else {
        for (size_t i = 0; i <= n; ++i) {
          if (i == ib) continue;
          for (size_t k = 0; k < n; ++k) s[i][k] = s[ib][k] + delta * (s[i][k] - s[ib][k]);
          fs[i] = F(s[i]);
        }
      }
    }
  }
  R.energy = F.best;
  R.x = F.best_x;
  R.n_evals = F.evals;
  return R;
}

OptimizeResult vqe_minimize(const Objective& f, std::vector<double> x0, Optimizer method,
                            const OptimizerOptions& opts) {
  return method == Optimizer::powell ? powell_minimize(f, std::move(x0), opts)
                                     : neldermead_minimize(f, std::move(x0), opts);
}

std::vector<double> parameter_shift_set(const std::vector<double>& th) {
  const size_t P = th.size();
  std::vector<double> rows;
  rows.reserve((1 + 2 * P) * P);
  rows.insert(rows.end(), th.begin(), th.end());
  const double h = 1.5707963267948966;
  for (size_t k = 0; k < P; ++k)
    for (double s : {h, -h}) {
      std::vector<double> r(th);
      r[k] += s;
      rows.insert(rows.end(), r.begin(), r.end());
    }
  return rows;
}

std::vector<double> exact_gradient_set(const std::vector<double>& th) {
  const size_t P = th.size();
  std::vector<double> rows(4 * P * P);
  const double shift[4] = {1.5707963267948966, -1.5707963267948966, 0.7853981633974483, -0.7853981633974483};
  for (size_t k = 0; k < P; ++k)
    for (size_t j = 0; j < 4; ++j) {
      double* r = rows.data() + (4 * k + j) * P;
      std::copy(th.begin(), th.end(), r);
      r[k] += shift[j];
    }
  return rows;
}

// dE/dt = c1 [E(+pi/2) - E(-pi/2)] + c2 [E(+pi/4) - E(-pi/4)],
// c1 = (1 - sqrt 2)/2, c2 = 1: exact for frequencies {1, 2}.
std::vector<double> exact_gradient_from_energies(const std::vector<double>& e, int P) {
  if ((int)e.size() != 4 * P) throw ContractViolation("exact_gradient_from_energies: need 4P energies");
  const double c1 = 0.5 * (1.0 - std::sqrt(2.0)), c2 = 1.0;
  std::vector<double> g((size_t)P);
  for (int k = 0; k < P; ++k)
    g[k] = c1 * (e[4 * k] - e[4 * k + 1]) + c2 * (e[4 * k + 2] - e[4 * k + 3]);
  return g;
}

namespace {
// BFGS on an energy and the 4P energies of exact_gradient_set(y) (in that row order)
OptimizeResult bfgs_core(const std::function<double(const std::vector<double>&)>& energy1,
                         const std::function<std::vector<double>(const std::vector<double>&)>& gradient_energies,
                         std::vector<double> x, const OptimizerOptions& opts) {
  const int P = (int)x.size();
  OptimizeResult R;
  auto energy = [&](const std::vector<double>& y) {
    ++R.n_evals;
    return energy1(y);
  };
  auto grad = [&](const std::vector<double>& y) {
    R.n_evals += 4 * P;
    return exact_gradient_from_energies(gradient_energies(y), P);
  };
  std::vector<double> Hinv((size_t)P * P, 0.0);
  for (int i = 0; i < P; ++i) Hinv[(size_t)i * P + i] = 1.0;
  double fx = energy(x);
  std::vector<double> g = grad(x);
  auto gmax = [&]() {
    double v = 0.0;
    for (double gi : g) v = std::max(v, std::abs(gi));
    return v;
  };
  bool reset_tried = false;  // a failed line search first retries steepest descent
  while (R.n_evals < opts.max_evals) {
    ++R.n_iterations;
    std::vector<double> d(P, 0.0);
    for (int i = 0; i < P; ++i)
      for (int j = 0; j < P; ++j) d[i] -= Hinv[(size_t)i * P + j] * g[j];
    double slope = 0.0;
    for (int i = 0; i < P; ++i) slope += d[i] * g[i];
    if (slope >= 0.0) {  // reset to steepest descent
      for (int i = 0; i < P; ++i) { d[i] = -g[i]; }
      std::fill(Hinv.begin(), Hinv.end(), 0.0);
      for (int i = 0; i < P; ++i) Hinv[(size_t)i * P + i] = 1.0;
      slope = 0.0;
      for (int i = 0; i < P; ++i) slope -= g[i] * g[i];
    }
    double t = 1.0, fn = fx;
    std::vector<double> xn(P);
    for (int ls = 0; ls < 40; ++ls) {
      for (int i = 0; i < P; ++i) xn[i] = x[i] + t * d[i];
      fn = energy(xn);
      if (fn <= fx + 1e-4 * t * slope) break;
      t *= 0.5;
    }
    if (!(fn < fx)) {
      // no decrease along d after 40 halvings: a stationary point within the
      // objective's resolution only if the gradient vanishes there; otherwise
      // restart from steepest descent once, then stop UNconverged
      if (gmax() <= 1e-6) { R.converged = true; break; }
      if (reset_tried) break;
      reset_tried = true;
      std::fill(Hinv.begin(), Hinv.end(), 0.0);
      for (int i = 0; i < P; ++i) Hinv[(size_t)i * P + i] = 1.0;
      continue;
    }
    reset_tried = false;
    std::vector<double> gn = grad(xn), s(P), y(P);
    for (int i = 0; i < P; ++i) { s[i] = xn[i] - x[i]; y[i] = gn[i] - g[i]; }
    const double df = fx - fn;
    x = xn; fx = fn; g = gn;
    // |dE| <= ftol on an accepted step, or a vanishing gradient
    if (df <= opts.ftol || gmax() <= 1e-6) { R.converged = true; break; }
    double sy = 0.0;
    for (int i = 0; i < P; ++i) sy += s[i] * y[i];
    if (sy > 1e-14) {
      std::vector<double> Hy(P, 0.0);
      for (int i = 0; i < P; ++i)
        for (int j = 0; j < P; ++j) Hy[i] += Hinv[(size_t)i * P + j] * y[j];
      double yHy = 0.0;
      for (int i = 0; i < P; ++i) yHy += y[i] * Hy[i];
      // (the two quotients once per update, not once per element: P^2 elements)
      const double a = (sy + yHy) / (sy * sy), b = 1.0 / sy;
      for (int i = 0; i < P; ++i) {
        const double as = a * s[i], bh = b * Hy[i], bs = b * s[i];
        double* row = &Hinv[(size_t)i * P];
        for (int j = 0; j < P; ++j) row[j] += as * s[j] - (bh * s[j] + bs * Hy[j]);
      }
    }
  }
  R.energy = fx;
  R.x = x;
  return R;
}
}  // namespace

OptimizeResult bfgs_minimize(const BatchObjective& f, std::vector<double> x, const OptimizerOptions& opts) {
  const int P = (int)x.size();
  return bfgs_core([&](const std::vector<double>& y) { return f(y, 1)[0]; },
                   [&](const std::vector<double>& y) { return f(exact_gradient_set(y), 4 * P); }, std::move(x), opts);
}

// ---- VQE loops on the device objective -------------------------------------------------
namespace {
// rows of amplitudes (generator order) -> energies, through the plan-order batch call
BatchObjective device_objective(Device& dev, const DevicePlan& plan, const DeviceHamiltonian& H, uint64_t hf) {
  return [&dev, &plan, &H, hf](const std::vector<double>& rows, int batch) {
    const std::vector<int>& order = plan.plan().order;
    const size_t P = order.size();
    if (rows.size() != P * (size_t)batch) throw ContractViolation("vqe: rows must be [batch][n_generators]");
    std::vector<double> th(rows.size());
    for (int b = 0; b < batch; ++b)
      for (size_t s = 0; s < P; ++s) th[(size_t)b * P + s] = rows[(size_t)b * P + (size_t)order[s]];
    return energy_batch(dev, plan, H, hf, th, batch);
  };
}
}  // namespace

OptimizeResult vqe_bfgs(Device& dev, const DevicePlan& plan, const DeviceHamiltonian& H, uint64_t hf,
                        std::vector<double> amps0, const OptimizerOptions& opts) {
  const std::vector<int>& order = plan.plan().order;
  const size_t P = order.size();
  if (amps0.size() != P) throw ContractViolation("vqe_bfgs: amplitude count mismatch");
  // bfgs_minimize on the device objective, with the 4P rows of a gradient call written
  // straight in plan order into one reused buffer: row (k, shift) is the permuted base
  // row with one entry changed, the same values device_objective(exact_gradient_set(y))
  // hands to the device (no 10 MB generator-order matrix and no permutation pass per call)
  std::vector<int> slot_of(P);  // generator k sits at plan position slot_of[k]
  for (size_t s = 0; s < P; ++s) slot_of[(size_t)order[s]] = (int)s;
  std::vector<double> base(P), rows(4 * P * P);
  const double shift[4] = {1.5707963267948966, -1.5707963267948966, 0.7853981633974483, -0.7853981633974483};
  const BatchObjective f1 = device_objective(dev, plan, H, hf);
  return bfgs_core(
      [&](const std::vector<double>& y) { return f1(y, 1)[0]; },
      [&](const std::vector<double>& y) {
        for (size_t s = 0; s < P; ++s) base[s] = y[(size_t)order[s]];
        auto fill = [&](size_t k0, size_t k1) {
          for (size_t k = k0; k < k1; ++k)
            for (size_t j = 0; j < 4; ++j) {
              double* r = rows.data() + (4 * k + j) * P;
              std::copy(base.begin(), base.end(), r);
              r[(size_t)slot_of[k]] = y[k] + shift[j];
            }
        };
        // (32 P^2 bytes per call: a few host threads when that is megabytes)
        const size_t nt = P >= 256 ? std::min<size_t>(4, std::max(1u, std::thread::hardware_concurrency())) : 1;
        std::vector<std::thread> th;
        for (size_t t = 1; t < nt; ++t) th.emplace_back(fill, P * t / nt, P * (t + 1) / nt);
        fill(0, P / nt);
        for (auto& t : th) t.join();
        return energy_batch(dev, plan, H, hf, rows, (int)(4 * P));
      },
      std::move(amps0), opts);
}

OptimizeResult vqe_device(Device& dev, const DevicePlan& plan, const DeviceHamiltonian& H, uint64_t hf,
                          std::vector<double> amps0, Optimizer method, const OptimizerOptions& opts) {
  if (amps0.size() != plan.plan().order.size()) throw ContractViolation("vqe_device: amplitude count mismatch");
  const BatchObjective f = device_objective(dev, plan, H, hf);
  return vqe_minimize([&f](const std::vector<double>& x) { return f(x, 1)[0]; }, std::move(amps0), method, opts);
}

// ---- FMO two-body assembly -----------------------------------------------------------
double assemble_two_body(int n_fragments, const std::map<std::string, double>& monomers,
                         const std::map<std::string, double>& dimers) {
  if ((int)monomers.size() != n_fragments)
    throw ContractViolation("assemble: expected " + std::to_string(n_fragments) +
                            " monomer energies, got " + std::to_string(monomers.size()));
  const size_t want = (size_t)n_fragments * (n_fragments - 1) / 2;
  if (dimers.size() != want)
    throw ContractViolation("assemble: expected " + std::to_string(want) + " dimer energies, got " +
                            std::to_string(dimers.size()));
  double e = 0.0, em = 0.0;
  for (auto& kv : dimers) e += kv.second;
  for (auto& kv : monomers) em += kv.second;
  return e - (n_fragments - 2) * em;
}

double FragmentLedger::assemble_corr() const { return assemble_two_body(n_fragments, corr_I, corr_IJ); }

double fragment_cost(const FragmentProblem& f) {
  std::map<uint64_t, int> groups;
  for (auto& kv : f.hamiltonian.terms()) groups[kv.first.first] = 1;
  return std::ldexp(1.0, f.plan.n_qubits) * (double)(f.plan.order.size() + groups.size());
}

std::vector<int> shard_by_cost(const std::vector<double>& costs, int world) {
  if (world < 1) throw ContractViolation("shard_by_cost: world must be >= 1");
  std::vector<int> idx(costs.size()), owner(costs.size(), 0);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return costs[a] > costs[b]; });
  std::vector<double> load((size_t)world, 0.0);
  for (int i : idx) {
    int best = 0;
    for (int r = 1; r < world; ++r)
      if (load[r] < load[best]) best = r;
    owner[i] = best;
    load[best] += costs[i];
  }
  return owner;
}

std::map<std::string, double> evaluate_fragments(Device& dev, const std::vector<FragmentProblem>& frags,
                                                 int rank, int world) {
  std::vector<double> costs;
  for (auto& f : frags) costs.push_back(fragment_cost(f));
  const std::vector<int> owner = shard_by_cost(costs, world);
  // this rank's fragments: upload, compile every device program on its own host
  // thread (ffq_energy_prepare is re-entrant for distinct plans), then evaluate
  std::vector<const FragmentProblem*> mine;
  for (size_t i = 0; i < frags.size(); ++i)
    if (owner[i] == rank) mine.push_back(&frags[i]);
  const bool dbg = std::getenv("FFQ_DEBUG") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!dbg) return;
    auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[ffq] evaluate_fragments %-10s %.1f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  std::vector<std::unique_ptr<DeviceHamiltonian>> Hs;
  std::vector<std::unique_ptr<DevicePlan>> Ps;
  for (const FragmentProblem* f : mine) {
    Hs.emplace_back(new DeviceHamiltonian(dev, f->hamiltonian));
    Ps.emplace_back(new DevicePlan(dev, f->plan));
  }
  lap("uploads");
  std::vector<std::thread> workers;
  std::vector<std::exception_ptr> errs(mine.size());
  for (size_t i = 0; i < mine.size(); ++i)
    workers.emplace_back([&, i] {
      try {
        prepare(dev, *Ps[i], *Hs[i], mine[i]->hf);
      } catch (...) {
        errs[i] = std::current_exception();
      }
    });
  for (auto& w : workers) w.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
  lap("compile");
  std::map<std::string, double> out;
  for (size_t i = 0; i < mine.size(); ++i)
    out[mine[i]->label] = energy_trotter(dev, mine[i]->amplitudes, *Ps[i], *Hs[i], mine[i]->hf) - mine[i]->e_reference;
  lap("energies");
  return out;
}

double assemble_fragments(int n_fragments, const std::map<std::string, double>& energies,
                          FragmentLedger* ledger) {
  FragmentLedger L;
  L.n_fragments = n_fragments;
  for (auto& kv : energies) (kv.first.size() == 1 ? L.corr_I : L.corr_IJ)[kv.first] = kv.second;
  const double e = L.assemble_corr();
  if (ledger) *ledger = L;
  return e;
}

std::vector<std::string> dimer_labels(int n_fragments) {
  std::vector<std::string> out;
  for (int j = 1; j <= n_fragments; ++j)
    for (int i = j + 1; i <= n_fragments; ++i) out.push_back(std::to_string(i) + std::to_string(j));
  return out;
}

}  // namespace fragfield
