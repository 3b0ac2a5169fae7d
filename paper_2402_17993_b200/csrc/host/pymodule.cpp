// pymodule.cpp -- pybind11 binding of the C++ operator API (include/fragfield)
// so tests and bench.py drive the same host code a C++ caller would. Every
// device call goes through the C-ABI in libfragfield_cuda.so.
#include <pybind11/complex.h>
#include <pybind11/functional.h>
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "fragfield/errors.hpp"
#include "fragfield/fmo_batch.hpp"
#include "fragfield/hamiltonian.hpp"
#include "fragfield/pauli.hpp"
#include "fragfield/statevector.hpp"
#include "fragfield/uccsd.hpp"
#include "fragfield/vqe.hpp"

namespace py = pybind11;
using namespace fragfield;

namespace {

using arr_u64 = py::array_t<uint64_t, py::array::c_style | py::array::forcecast>;
using arr_f64 = py::array_t<double, py::array::c_style | py::array::forcecast>;
using arr_c128 = py::array_t<std::complex<double>, py::array::c_style | py::array::forcecast>;

py::tuple psum_arrays(const PauliSum& s) {
  std::vector<uint64_t> x, z;
  std::vector<double> re, im;
  s.flatten(x, z, re, im);
  arr_u64 X(x.size()), Z(z.size());
  arr_c128 C(re.size());
  for (size_t i = 0; i < x.size(); ++i) {
    X.mutable_at(i) = x[i];
    Z.mutable_at(i) = z[i];
    C.mutable_at(i) = {re[i], im[i]};
  }
  return py::make_tuple(X, Z, C);
}

PauliSum psum_from_arrays(int n, arr_u64 x, arr_u64 z, arr_c128 c) {
  PauliSum s(n);
  if (x.size() != z.size() || x.size() != c.size()) throw ContractViolation("term arrays differ in length");
  for (py::ssize_t i = 0; i < x.size(); ++i) s.add(x.at(i), z.at(i), c.at(i));
  s.simplify();
  return s;
}

std::vector<double> to_vec(arr_f64 a) { return std::vector<double>(a.data(), a.data() + a.size()); }

}  // namespace

PYBIND11_MODULE(_fragfield, m) {
  m.doc() = "fragfield B200 UCCSD hot path: host operator API over libfragfield_cuda.so";

  py::register_exception<ContractViolation>(m, "ContractViolation", PyExc_ValueError);
  py::register_exception<DeviceError>(m, "DeviceError", PyExc_RuntimeError);
  py::register_exception<ConvergenceError>(m, "ConvergenceError", PyExc_RuntimeError);
  py::register_exception<ParseError>(m, "ParseError", PyExc_ValueError);

  // ---- qubit-map ----
  py::class_<PauliString>(m, "PauliString")
      .def(py::init([](int n, uint64_t x, uint64_t z) { return PauliString{n, x, z}; }),
           py::arg("n_qubits"), py::arg("x") = 0, py::arg("z") = 0)
      .def_readonly("n_qubits", &PauliString::n_qubits)
      .def_readonly("x", &PauliString::x)
      .def_readonly("z", &PauliString::z)
      .def("letters", &PauliString::letters)
      .def_static("parse", &PauliString::parse)
      .def("__repr__", [](const PauliString& p) { return "PauliString('" + p.letters() + "')"; });
  m.def("pauli_mul", &pauli_mul);

  py::class_<PauliSum>(m, "PauliSum")
      .def(py::init<int>(), py::arg("n_qubits"))
      .def_static("from_arrays", &psum_from_arrays)
      .def_static("from_text", &PauliSum::from_text)
      .def_property_readonly("n_qubits", &PauliSum::n_qubits)
      .def("add", [](PauliSum& s, const PauliString& p, Complex c) { s.add(p, c); })
      .def("simplify", &PauliSum::simplify, py::arg("tol") = 1e-14)
      .def("arrays", &psum_arrays)
      .def("to_text", &PauliSum::to_text)
      .def("is_hermitian", &PauliSum::is_hermitian, py::arg("tol") = 1e-12)
      .def("is_antihermitian", &PauliSum::is_antihermitian, py::arg("tol") = 1e-12)
      .def("__len__", &PauliSum::size)
      .def("__add__", &PauliSum::operator+)
      .def("__mul__", &PauliSum::operator*)
      .def_property_readonly("n_qubits", &PauliSum::n_qubits);

  m.def(
      "jordan_wigner",
      [](const std::vector<std::pair<Complex, std::vector<std::pair<int, bool>>>>& terms, int n_so) {
        FermionOperator op;
        for (auto& t : terms) {
          FermionTerm ft{t.first, {}};
          for (auto& o : t.second) ft.ops.push_back({o.first, o.second});
          op.push_back(ft);
        }
        return jordan_wigner(op, n_so);
      },
      py::arg("terms"), py::arg("n_so"),
      "terms: [(coef, [(index, is_dagger), ...]), ...], operator products left to right");

  // ---- hamiltonian ----
  m.def(
      "synthetic_integrals",
      [](int mo, uint64_t seed, double sh, double sg) {
        SpatialIntegrals I = synthetic_integrals(mo, seed, sh, sg);
        arr_f64 h({mo, mo}), g({mo, mo, mo, mo});
        std::copy(I.h.begin(), I.h.end(), h.mutable_data());
        std::copy(I.g.begin(), I.g.end(), g.mutable_data());
        return py::make_tuple(h, g);
      },
      py::arg("m"), py::arg("seed"), py::arg("sigma_h") = 1.0, py::arg("sigma_g") = 0.1);
  m.def(
      "qubit_hamiltonian",
      [](arr_f64 h, arr_f64 g, int n_elec, double e_const) {
        SpatialIntegrals I;
        I.m = (int)h.shape(0);
        I.h = to_vec(h);
        I.g = to_vec(g);
        I.e_const = e_const;
        if (I.h.size() != (size_t)I.m * I.m || I.g.size() != (size_t)I.m * I.m * I.m * I.m)
          throw ContractViolation("qubit_hamiltonian: integral shapes");
        return qubit_hamiltonian(to_spin_orbitals(I, n_elec));
      },
      py::arg("h"), py::arg("g"), py::arg("n_elec"), py::arg("e_const") = 0.0);
  m.def(
      "ao_to_mo",
      [](arr_f64 h, arr_f64 g, arr_f64 C, double e_const, py::object v_esp) {
        SpatialIntegrals I;
        I.m = (int)h.shape(0);
        I.h = to_vec(h);
        I.g = to_vec(g);
        I.e_const = e_const;
        const int mo = C.ndim() == 2 ? (int)C.shape(1) : 0;
        std::vector<double> v;
        if (!v_esp.is_none()) v = to_vec(v_esp.cast<arr_f64>());
        SpatialIntegrals R = ao_to_mo(I, to_vec(C), mo, v);
        arr_f64 ho({mo, mo}), go({mo, mo, mo, mo});
        std::copy(R.h.begin(), R.h.end(), ho.mutable_data());
        std::copy(R.g.begin(), R.g.end(), go.mutable_data());
        return py::make_tuple(ho, go, R.e_const);
      },
      py::arg("h"), py::arg("g"), py::arg("C"), py::arg("e_const") = 0.0, py::arg("v_esp") = py::none(),
      "SPEC.md:272-279 -> (h_mo, g_mo, e_const)");
  m.def(
      "freeze_core",
      [](arr_f64 h, arr_f64 g, double e_const, int n_frozen, int n_elec) {
        SpatialIntegrals I;
        I.m = (int)h.shape(0);
        I.h = to_vec(h);
        I.g = to_vec(g);
        I.e_const = e_const;
        if (I.h.size() != (size_t)I.m * I.m || I.g.size() != (size_t)I.m * I.m * I.m * I.m)
          throw ContractViolation("freeze_core: integral shapes");
        FrozenCore F = freeze_core(I, n_frozen, n_elec);
        const int ma = F.active.m;
        arr_f64 ho({ma, ma}), go({ma, ma, ma, ma});
        std::copy(F.active.h.begin(), F.active.h.end(), ho.mutable_data());
        std::copy(F.active.g.begin(), F.active.g.end(), go.mutable_data());
        return py::make_tuple(ho, go, F.active.e_const, F.e_frozen, F.n_elec_active);
      },
      py::arg("h"), py::arg("g"), py::arg("e_const"), py::arg("n_frozen"), py::arg("n_elec"),
      "SPEC.md:280-289 -> (h_eff, g_active, e_const incl. E_frozen, E_frozen, active electrons)");
  m.def("random_pauli_hamiltonian", &random_pauli_hamiltonian, py::arg("n_qubits"),
        py::arg("n_terms"), py::arg("seed"), py::arg("sigma") = 0.1);
  m.def("uniform_vector", &uniform_vector);
  m.def(
      "write_fcidump",
      [](const std::string& path, arr_f64 h, arr_f64 g, int n_elec, double e_const, int ms2) {
        SpatialIntegrals I;
        I.m = (int)h.shape(0);
        I.h = to_vec(h);
        I.g = to_vec(g);
        I.e_const = e_const;
        write_fcidump(path, I, n_elec, ms2);
      },
      py::arg("path"), py::arg("h"), py::arg("g"), py::arg("n_elec"), py::arg("e_const") = 0.0,
      py::arg("ms2") = 0);
  m.def(
      "read_fcidump",
      [](const std::string& path) {
        Fcidump F = read_fcidump(path);
        const int mo = F.ints.m;
        arr_f64 h({mo, mo}), g({mo, mo, mo, mo});
        std::copy(F.ints.h.begin(), F.ints.h.end(), h.mutable_data());
        std::copy(F.ints.g.begin(), F.ints.g.end(), g.mutable_data());
        return py::make_tuple(h, g, F.ints.e_const, F.n_elec, F.ms2);
      },
      py::arg("path"), "-> (h, g, e_const, n_elec, ms2)");
  m.def("write_state_dump", &write_state_dump, py::arg("path"), py::arg("n_qubits"), py::arg("amplitudes"));
  m.def(
      "read_state_dump",
      [](const std::string& path) {
        int n = 0;
        auto a = read_state_dump(path, &n);
        return py::make_tuple(n, a);
      },
      py::arg("path"), "-> (n_qubits, amplitudes)");
  m.def("reduce_two_qubits", &reduce_two_qubits, py::arg("op"), py::arg("n_so"), py::arg("n_alpha"),
        py::arg("n_beta"));
  m.def("reduce_two_qubits_basis", &reduce_two_qubits_basis, py::arg("jw_bits"), py::arg("n_so"));

  // ---- uccsd ----
  py::class_<Excitation>(m, "Excitation")
      .def_readonly("kind", &Excitation::kind)
      .def_readonly("i", &Excitation::i)
      .def_readonly("j", &Excitation::j)
      .def_readonly("a", &Excitation::a)
      .def_readonly("b", &Excitation::b);
  py::class_<Generator>(m, "Generator")
      .def_readonly("id", &Generator::id)
      .def_readonly("exc", &Generator::exc)
      .def_readonly("image", &Generator::image);
  m.def("build_generators", &build_generators, py::arg("n_so"), py::arg("n_elec"));
  py::class_<TrotterPlan>(m, "TrotterPlan")
      .def_readonly("n_qubits", &TrotterPlan::n_qubits)
      .def_readonly("order", &TrotterPlan::order)
      .def_readonly("generators", &TrotterPlan::generators)
      .def("plan_theta", &TrotterPlan::plan_theta);
  m.def("magnitude_order", &magnitude_order, py::arg("generators"), py::arg("amplitudes"),
        py::arg("n_qubits"));
  m.def("hf_bits", &hf_bits);

  // ---- device (C-ABI) ----
  py::class_<Device>(m, "Device")
      .def(py::init<int>(), py::arg("ordinal") = 0)
      .def_property_readonly("ordinal", &Device::ordinal)
      .def("kernel_launches", &Device::kernel_launches)
      .def("synchronize", &Device::synchronize)
      .def_static("count", &Device::count);
  py::class_<DeviceHamiltonian>(m, "DeviceHamiltonian")
      .def(py::init<Device&, const PauliSum&>(), py::keep_alive<1, 2>())
      .def_property_readonly("n_groups", &DeviceHamiltonian::n_groups)
      .def_property_readonly("n_classes", &DeviceHamiltonian::n_classes)
      .def_property_readonly("n_qubits", &DeviceHamiltonian::n_qubits);
  py::class_<DevicePlan>(m, "DevicePlan")
      .def(py::init<Device&, const TrotterPlan&>(), py::keep_alive<1, 2>())
      .def_property_readonly("n_fused", &DevicePlan::n_fused)
      .def_property_readonly("n_string_ops", &DevicePlan::n_string_ops)
      .def_property_readonly("plan", &DevicePlan::plan);
  py::class_<Statevector>(m, "Statevector")
      .def(py::init<Device&, int, int>(), py::keep_alive<1, 2>(), py::arg("device"),
           py::arg("n_qubits"), py::arg("batch") = 1)
      .def("set_basis", &Statevector::set_basis)
      .def("apply_pauli_rotation", &Statevector::apply_pauli_rotation)
      .def("apply_plan", [](Statevector& s, const DevicePlan& p, arr_f64 th) { s.apply_plan(p, to_vec(th)); })
      .def("expectation", &Statevector::expectation)
      .def("download",
           [](const Statevector& s) {
             auto v = s.download();
             arr_c128 out({(py::ssize_t)s.batch(), (py::ssize_t)1 << s.n_qubits()});
             std::copy(v.begin(), v.end(), out.mutable_data());
             return out;
           })
      .def("upload", [](Statevector& s, arr_c128 a) {
        s.upload(std::vector<Complex>(a.data(), a.data() + a.size()));
      });
  m.def(
      "energy_batch",
      [](Device& dev, const DevicePlan& plan, const DeviceHamiltonian& H, uint64_t hf, arr_f64 theta) {
        const size_t ng = plan.plan().order.size();
        const int batch = ng ? (int)(theta.size() / ng) : (int)theta.shape(0);
        auto e = energy_batch(dev, plan, H, hf, to_vec(theta), batch);
        arr_f64 out(e.size());
        std::copy(e.begin(), e.end(), out.mutable_data());
        return out;
      },
      py::arg("device"), py::arg("plan"), py::arg("hamiltonian"), py::arg("hf_bits"), py::arg("theta"));
  m.def("energy_trotter", &energy_trotter);
  m.def("energy_exact", &energy_exact, py::arg("device"), py::arg("amplitudes"), py::arg("plan"),
        py::arg("hamiltonian"), py::arg("hf_bits"), py::arg("tol") = 1e-12);
  py::class_<GroundState>(m, "GroundState")
      .def_readonly("energy", &GroundState::energy)
      .def_readonly("iterations", &GroundState::iterations)
      .def_readonly("dimension", &GroundState::dimension);
  m.def("lanczos_ground", &lanczos_ground, py::arg("device"), py::arg("hamiltonian"), py::arg("hf_bits"),
        py::arg("tol") = 1e-10, py::arg("max_iter") = 500);

  // ---- vqe ----
  py::class_<OptimizerOptions>(m, "OptimizerOptions")
      .def(py::init<>())
      .def_readwrite("ftol", &OptimizerOptions::ftol)
      .def_readwrite("max_evals", &OptimizerOptions::max_evals)
      .def_readwrite("xtol", &OptimizerOptions::xtol)
      .def_readwrite("initial_step", &OptimizerOptions::initial_step);
  py::class_<OptimizeResult>(m, "OptimizeResult")
      .def_readonly("energy", &OptimizeResult::energy)
      .def_readonly("x", &OptimizeResult::x)
      .def_readonly("n_evals", &OptimizeResult::n_evals)
      .def_readonly("n_iterations", &OptimizeResult::n_iterations)
      .def_readonly("converged", &OptimizeResult::converged);
  m.def("powell_minimize", &powell_minimize, py::arg("f"), py::arg("x0"), py::arg("opts") = OptimizerOptions{});
  m.def("neldermead_minimize", &neldermead_minimize, py::arg("f"), py::arg("x0"),
        py::arg("opts") = OptimizerOptions{});
  m.def("bfgs_minimize", &bfgs_minimize, py::arg("f"), py::arg("x0"), py::arg("opts") = OptimizerOptions{});
  m.def("vqe_bfgs", &vqe_bfgs, py::arg("device"), py::arg("plan"), py::arg("hamiltonian"), py::arg("hf_bits"),
        py::arg("amplitudes"), py::arg("opts") = OptimizerOptions{}, py::call_guard<py::gil_scoped_release>());
  m.def(
      "vqe_device",
      [](Device& dev, const DevicePlan& plan, const DeviceHamiltonian& H, uint64_t hf, std::vector<double> x0,
         const std::string& method, const OptimizerOptions& opts) {
        if (method != "powell" && method != "neldermead") throw ContractViolation("vqe_device: unknown optimizer");
        py::gil_scoped_release nogil;
        return vqe_device(dev, plan, H, hf, std::move(x0),
                          method == "powell" ? Optimizer::powell : Optimizer::neldermead, opts);
      },
      py::arg("device"), py::arg("plan"), py::arg("hamiltonian"), py::arg("hf_bits"), py::arg("amplitudes"),
      py::arg("method") = "powell", py::arg("opts") = OptimizerOptions{});
  m.def("parameter_shift_set", &parameter_shift_set);
  m.def("exact_gradient_set", &exact_gradient_set);
  m.def("exact_gradient_from_energies", &exact_gradient_from_energies);

  // ---- FMO ----
  m.def("assemble_two_body", &assemble_two_body);
  m.def("dimer_labels", &dimer_labels);
  py::class_<FragmentProblem>(m, "FragmentProblem")
      .def(py::init([](std::string label, const PauliSum& H, const TrotterPlan& plan, uint64_t hf,
                       std::vector<double> amps, double e_ref) {
             return FragmentProblem{std::move(label), H, plan, hf, std::move(amps), e_ref};
           }),
           py::arg("label"), py::arg("hamiltonian"), py::arg("plan"), py::arg("hf"), py::arg("amplitudes"),
           py::arg("e_reference") = 0.0)
      .def_readonly("label", &FragmentProblem::label)
      .def_readonly("hf", &FragmentProblem::hf)
      .def_readonly("amplitudes", &FragmentProblem::amplitudes);
  m.def("fragment_cost", &fragment_cost);
  m.def("shard_by_cost", &shard_by_cost, py::arg("costs"), py::arg("world"));
  m.def("evaluate_fragments", &evaluate_fragments, py::arg("device"), py::arg("fragments"),
        py::arg("rank") = 0, py::arg("world") = 1);
  m.def("assemble_fragments",
        [](int nf, const std::map<std::string, double>& e) { return assemble_fragments(nf, e, nullptr); });
}
