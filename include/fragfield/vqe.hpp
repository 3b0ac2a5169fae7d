// fragfield/vqe.hpp -- VQE drivers around the batched energy:
// derivative-free Powell and Nelder-Mead, plus gradient sets (parameter-shift
// workload of BASELINE.json config 2 and the exact four-term rule for UCCSD
// generators) and a BFGS driver that consumes batched gradients (config 3).
#pragma once

#include <functional>
#include <vector>

namespace fragfield {

struct OptimizerOptions {
  double ftol = 1e-8;       // |dE| convergence, Hartree
  int max_evals = 20000;
  double xtol = 1e-10;
  double initial_step = 0.1;
};

struct OptimizeResult {
  double energy = 0.0;
  std::vector<double> x;
  int n_evals = 0;
  int n_iterations = 0;
  bool converged = false;
};

using Objective = std::function<double(const std::vector<double>&)>;
/// Batched objective: f(X) for rows X[b*dim .. b*dim+dim) -> energies[b].
using BatchObjective = std::function<std::vector<double>(const std::vector<double>&, int)>;

OptimizeResult powell_minimize(const Objective& f, std::vector<double> x0,
                               const OptimizerOptions& opts = {});
OptimizeResult neldermead_minimize(const Objective& f, std::vector<double> x0,
                                   const OptimizerOptions& opts = {});
enum class Optimizer { powell, neldermead };
OptimizeResult vqe_minimize(const Objective& f, std::vector<double> x0, Optimizer method,
                            const OptimizerOptions& opts = {});

/// Config-2 workload definition: rows [theta, theta + pi/2 e_k, theta - pi/2 e_k]
/// for k = 0..P-1 (1 + 2P rows, k-major).
std::vector<double> parameter_shift_set(const std::vector<double>& theta);
/// Exact gradient rule for generators whose energy has frequencies {1, 2}
/// (every UCCSD excitation): shifts (+-pi/2, +-pi/4), 4P rows.
std::vector<double> exact_gradient_set(const std::vector<double>& theta);
std::vector<double> exact_gradient_from_energies(const std::vector<double>& e, int P);

/// BFGS with the batched exact gradient (one batched call per iteration).
OptimizeResult bfgs_minimize(const BatchObjective& f, std::vector<double> x0,
                             const OptimizerOptions& opts = {});

class Device;
class DevicePlan;
class DeviceHamiltonian;

/// The VQE loop of SPEC.md:525-541 with the device objective built in: amplitudes
/// in generator order, every energy through energy_batch on `dev` (no
/// host-language callback inside the loop). vqe_bfgs runs bfgs_minimize with one
/// batched 4P-row gradient call per iteration; vqe_device runs the serial
/// Powell / Nelder-Mead optimizers on the B = 1 path.
OptimizeResult vqe_bfgs(Device& dev, const DevicePlan& plan, const DeviceHamiltonian& H, uint64_t hf,
                        std::vector<double> amps0, const OptimizerOptions& opts = {});
OptimizeResult vqe_device(Device& dev, const DevicePlan& plan, const DeviceHamiltonian& H, uint64_t hf,
                          std::vector<double> amps0, Optimizer method, const OptimizerOptions& opts = {});

}  // namespace fragfield
