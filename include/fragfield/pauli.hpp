// fragfield/pauli.hpp -- qubit-map module: packed Pauli
// strings, Pauli sums with canonical ordering, and the Jordan-Wigner map.
#pragma once

#include <complex>
#include <cstdint>
#include <map>
#include <string>
#include <utility>
#include <vector>

namespace fragfield {

using Complex = std::complex<double>;

/// Phase-free Pauli string over n qubits. Bit q of x / z:
/// X if only x, Z if only z, Y if both. Qubit 0 = least significant bit.
struct PauliString {
  int n_qubits = 0;
  uint64_t x = 0, z = 0;
  bool operator<(const PauliString& o) const {
    return x != o.x ? x < o.x : z < o.z;  // canonical order
  }
  bool operator==(const PauliString& o) const { return x == o.x && z == o.z && n_qubits == o.n_qubits; }
  /// Letters with qubit 0 first (pinned text convention).
  std::string letters() const;
  static PauliString parse(const std::string& letters);
};

/// Product A*B = i^k C. Returns (k, C).
std::pair<int, PauliString> pauli_mul(const PauliString& a, const PauliString& b);

/// Map PauliString -> complex coefficient, canonical order, no zero entries
/// after simplify.
class PauliSum {
 public:
  explicit PauliSum(int n_qubits = 0) : n_(n_qubits) {}
  int n_qubits() const { return n_; }
  void add(uint64_t x, uint64_t z, Complex c);
  void add(const PauliString& p, Complex c) { add(p.x, p.z, c); }
  /// Drops |c| <= tol (the pinned simplify threshold is 1e-14).
  void simplify(double tol = 1e-14);
  size_t size() const { return terms_.size(); }
  const std::map<std::pair<uint64_t, uint64_t>, Complex>& terms() const { return terms_; }
  PauliSum operator+(const PauliSum& o) const;
  PauliSum operator*(const PauliSum& o) const;
  PauliSum scaled(Complex s) const;
  /// Flat arrays in canonical order (for the C-ABI).
  void flatten(std::vector<uint64_t>& x, std::vector<uint64_t>& z, std::vector<double>& re,
               std::vector<double>& im) const;
  /// One term per line: "coeff_re coeff_im letters".
  std::string to_text() const;
  static PauliSum from_text(const std::string& text);
  bool is_hermitian(double tol = 1e-12) const;
  bool is_antihermitian(double tol = 1e-12) const;

 private:
  int n_;
  std::map<std::pair<uint64_t, uint64_t>, Complex> terms_;
};

/// a_p (dagger=false) or a+_p (dagger=true)
struct LadderOp {
  int index;
  bool dagger;
};
struct FermionTerm {
  Complex coef;
  std::vector<LadderOp> ops;  // operator product as written, left to right
};
using FermionOperator = std::vector<FermionTerm>;

/// a+_p -> 1/2 (X_p - i Y_p) Z_{p-1}..Z_0. Throws
/// ContractViolation on an index >= n_so.
PauliSum jordan_wigner(const FermionOperator& op, int n_so);
PauliSum jordan_wigner_ladder(const LadderOp& op, int n_so);

/// reduce_two_qubits: the symmetry-conserving two-qubit
/// reduction of a JW-mapped (interleaved alpha/beta) operator.
/// Modes are re-ordered alpha first (spin orbital 2P -> P, 2P+1 -> m + P,
/// m = n_so / 2) and parity-encoded: qubit j holds the parity of modes
/// 0..j. This is the GF(2)-linear basis change y = A x of occupation bits x,
/// so X^a Z^b -> X^(A a) Z^(A^-T b) (phases from Y = iXZ carried exactly).
/// Qubit m - 1 then holds the N_alpha parity and qubit n_so - 1 the N parity;
/// both are replaced by their eigenvalues for (n_alpha, n_beta) and removed,
/// leaving n_so - 2 qubits (pinned layout; SPEC leaves the ordering open).
/// Throws ContractViolation when a term acts with X or Y on a tapered qubit
/// (the operator does not conserve the two parities).
PauliSum reduce_two_qubits(const PauliSum& op, int n_so, int n_alpha, int n_beta);
/// The same reduction of a JW occupation bitstring (e.g. |HF>).
uint64_t reduce_two_qubits_basis(uint64_t jw_bits, int n_so);

}  // namespace fragfield
