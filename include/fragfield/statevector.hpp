// fragfield/statevector.hpp -- device-resident simulator and batched energy
// evaluation, a thin RAII facade over the C-ABI in
// fragfield_cuda.h. Every object here lives on one B200; there is no CPU
// fallback (a missing device raises DeviceError).
#pragma once

#include <complex>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "fragfield/errors.hpp"
#include "fragfield/pauli.hpp"
#include "fragfield/uccsd.hpp"
#include "fragfield_cuda.h"

namespace fragfield {

/// State dump: little-endian int64 n_qubits, then 2^n complex
/// doubles (re, im) in natural binary order, qubit 0 = least significant bit.
void write_state_dump(const std::string& path, int n_qubits, const std::vector<std::complex<double>>& amps);
std::vector<std::complex<double>> read_state_dump(const std::string& path, int* n_qubits);

/// Throws ContractViolation (FFQ_EINVAL, FFQ_ENONHERMITIAN) or DeviceError.
void check_ffq(int rc, ffq_ctx_t ctx);

class Device {
 public:
  explicit Device(int ordinal = 0);
  ~Device();
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  ffq_ctx_t handle() const { return ctx_; }
  int ordinal() const { return ordinal_; }
  int64_t kernel_launches() const { return ffq_ctx_kernel_launches(ctx_); }
  void synchronize() const;
  static int count();

 private:
  ffq_ctx_t ctx_ = nullptr;
  int ordinal_ = 0;
};

/// Grouped, device-resident qubit Hamiltonian (immutable after upload).
class DeviceHamiltonian {
 public:
  DeviceHamiltonian(Device& dev, const PauliSum& H);
  ~DeviceHamiltonian();
  DeviceHamiltonian(const DeviceHamiltonian&) = delete;
  DeviceHamiltonian& operator=(const DeviceHamiltonian&) = delete;
  ffq_ham_t handle() const { return h_; }
  int n_qubits() const { return n_; }
  int n_groups() const;
  int64_t n_classes() const;

 private:
  Device& dev_;
  ffq_ham_t h_ = nullptr;
  int n_ = 0;
};

/// Device copy of a TrotterPlan (generators fused into exact rotation passes).
class DevicePlan {
 public:
  DevicePlan(Device& dev, const TrotterPlan& plan);
  ~DevicePlan();
  DevicePlan(const DevicePlan&) = delete;
  DevicePlan& operator=(const DevicePlan&) = delete;
  ffq_plan_t handle() const { return p_; }
  const TrotterPlan& plan() const { return plan_; }
  int n_fused() const;
  int n_string_ops() const;

 private:
  Device& dev_;
  ffq_plan_t p_ = nullptr;
  TrotterPlan plan_;
};

/// A batch of state vectors [batch][2^n] complex128 on the device.
class Statevector {
 public:
  Statevector(Device& dev, int n_qubits, int batch = 1);
  ~Statevector();
  Statevector(const Statevector&) = delete;
  Statevector& operator=(const Statevector&) = delete;
  int n_qubits() const { return n_; }
  int batch() const { return batch_; }
  /// hf_state: every row becomes |bits>.
  void set_basis(uint64_t bits);
  /// e^{i theta P} on every row.
  void apply_pauli_rotation(const PauliString& p, double theta);
  /// e^{i theta_r P_r} for r = 0, 1, ... in order; runs of low-qubit flip
  /// masks are applied per shared-memory tile (ffq_state_apply_pauli_rotations).
  void apply_pauli_rotations(const std::vector<PauliString>& ps, const std::vector<double>& theta);
  /// theta [batch][n_gen] in plan order.
  void apply_plan(const DevicePlan& plan, const std::vector<double>& theta);
  /// <psi|H|psi> per row; throws ContractViolation if |Im| > 1e-10.
  std::vector<double> expectation(const DeviceHamiltonian& H) const;
  std::vector<Complex> download() const;
  void upload(const std::vector<Complex>& amps);

 private:
  Device& dev_;
  ffq_state_t s_ = nullptr;
  int n_, batch_;
};

/// Compile and cache the device program of (plan, H, hf) ahead of the first
/// energy call (ffq_energy_prepare); safe to call from several host threads for
/// distinct plans of one device.
void prepare(Device& dev, const DevicePlan& plan, const DeviceHamiltonian& H, uint64_t hf);

/// energy_trotter for a batch of amplitude vectors given in
/// plan order: e[b] = <HF| U(theta_b)^dag H U(theta_b) |HF>.
std::vector<double> energy_batch(Device& dev, const DevicePlan& plan, const DeviceHamiltonian& H,
                                 uint64_t hf, const std::vector<double>& theta_plan_order,
                                 int batch);

/// Single evaluation with amplitudes indexed by canonical generator id.
double energy_trotter(Device& dev, const std::vector<double>& amps, const DevicePlan& plan,
                      const DeviceHamiltonian& H, uint64_t hf);

/// Trotter-free UCCSD energy, amplitudes by canonical id.
double energy_exact(Device& dev, const std::vector<double>& amps, const DevicePlan& plan,
                    const DeviceHamiltonian& H, uint64_t hf, double tol = 1e-12);

/// CAS-CI ground energy in the Krylov space of |hf>.
struct GroundState {
  double energy = 0.0;
  int iterations = 0, dimension = 0;
};
GroundState lanczos_ground(Device& dev, const DeviceHamiltonian& H, uint64_t hf, double tol = 1e-10,
                           int max_iter = 500);

}  // namespace fragfield
