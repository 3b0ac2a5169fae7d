"""SURVEY 8f2 on the GPU: lanczos_ground (CAS-CI in the HF sector) and the
Trotter-free energy_exact, checked against dense numpy/scipy references and the
SPEC invariants (single-generator Trotter = exact; variational
bound)."""
import numpy as np
import pytest
import scipy.linalg as sl

from dense import ladder_dense, pauli_dense
from paper_2402_17993_b200 import capi, problems

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return capi.Context(0)


def sector_matrix(P):
    """Dense H restricted to the (N_alpha, N_beta) sector of |HF> (numpy)."""
    n = P.n_qubits
    na = bin(P.hf & int("01" * (n // 2), 2)).count("1")
    nb = bin(P.hf & int("10" * (n // 2), 2)).count("1")
    ks = [k for k in range(1 << n) if bin(k & int("01" * (n // 2), 2)).count("1") == na
          and bin(k & int("10" * (n // 2), 2)).count("1") == nb]
    pos = {k: i for i, k in enumerate(ks)}
    M = np.zeros((len(ks), len(ks)), complex)
    x, z, c = P.ham_arrays()
    for xx, zz, cc in zip(x.astype(int), z.astype(int), c):
        ny = bin(xx & zz).count("1")
        for k in ks:
            kp = k ^ xx
            if kp in pos:
                M[pos[kp], pos[k]] += cc * (1j ** ny) * (-1) ** bin(k & zz).count("1")
    return M, ks


@pytest.mark.parametrize("config", [1, 2])
def test_lanczos_ground_vs_dense_sector(ctx, config):
    P = problems.config_problem(config)
    ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
    e0, iters, dim = capi.lanczos_ground(ctx, ham, P.hf, tol=1e-12)
    M, ks = sector_matrix(P)
    assert dim == len(ks)
    assert abs(e0 - np.linalg.eigvalsh(M)[0]) <= 1e-9


def test_energy_exact_vs_dense_expm_and_single_generator(ctx):
    P = problems.config_problem(1)
    n = P.n_qubits
    plan = capi.Plan(ctx, n, *P.plan_arrays())
    ham = capi.Hamiltonian(ctx, n, *P.ham_arrays())
    th = P.plan_thetas()[0]
    e = capi.energy_exact(ctx, plan, ham, P.hf, th)
    # dense: exp(sum_g t_g (tau_g - tau_g^dag)) |HF>
    a = [ladder_dense(n, p, False) for p in range(n)]
    ad = [ladder_dense(n, p, True) for p in range(n)]
    A = np.zeros((1 << n, 1 << n))
    for gen, t in zip(P.gens, P.thetas[0]):
        ex = gen.exc
        tau = ad[ex.a] @ a[ex.i] if ex.kind == 1 else ad[ex.a] @ ad[ex.b] @ a[ex.j] @ a[ex.i]
        A += t * (tau - tau.T)
    v = np.zeros(1 << n)
    v[P.hf] = 1.0
    v = sl.expm(A) @ v
    x, z, c = P.ham_arrays()
    H = sum(cc * pauli_dense(n, xx, zz) for xx, zz, cc in zip(x, z, c))
    assert abs(e - np.vdot(v, H @ v).real) <= 1e-10
    # one generator: Trotterization is exact
    one = np.zeros_like(th)
    one[0] = 0.37
    e_tr = capi.energy_batch(ctx, plan, ham, P.hf, one[None, :])[0]
    assert abs(capi.energy_exact(ctx, plan, ham, P.hf, one) - e_tr) <= 1e-12
    # zero amplitudes: HF energy
    assert abs(capi.energy_exact(ctx, plan, ham, P.hf, np.zeros_like(th)) -
               capi.energy_batch(ctx, plan, ham, P.hf, np.zeros((1, len(th))))[0]) <= 1e-12


def test_variational_bound_18q(ctx):
    # every UCCSD energy (Trotterized or exact) >= E_CASCI - 1e-10
    P = problems.config_problem(3, batch=8)
    plan = capi.Plan(ctx, P.n_qubits, *P.plan_arrays())
    ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
    e0, iters, dim = capi.lanczos_ground(ctx, ham, P.hf, tol=1e-10)
    assert dim == 15876
    e = capi.energy_batch(ctx, plan, ham, P.hf, P.plan_thetas())
    assert np.all(e >= e0 - 1e-10)
    ex = capi.energy_exact(ctx, plan, ham, P.hf, P.plan_thetas()[0])
    assert ex >= e0 - 1e-10
    print(f"E_CASCI = {e0:.10f} ({iters} Lanczos iterations), Trotter {e[0]:.10f}, exact {ex:.10f}")


def test_cpp_facade_exact_references():
    import paper_2402_17993_b200 as ff

    dev = ff.Device(0)
    P = problems.config_problem(1)
    H = ff.DeviceHamiltonian(dev, P.H)
    plan = ff.DevicePlan(dev, P.plan)
    g = ff.lanczos_ground(dev, H, P.hf)
    e_tr = ff.energy_trotter(dev, list(P.thetas[0]), plan, H, P.hf)
    e_ex = ff.energy_exact(dev, list(P.thetas[0]), plan, H, P.hf)
    assert g.dimension == 36 and e_tr >= g.energy - 1e-10 and e_ex >= g.energy - 1e-10


def test_config2_vqe_converges_to_ftol_and_is_variational():
    """BASELINE config 2 (12 qubits): BFGS on batched exact gradients through
    the C-ABI converges to ftol 1e-8 (|dE| of an accepted step)
    below the HF energy and above E_CASCI - 1e-10."""
    import paper_2402_17993_b200 as ff

    P = problems.config_problem(2)
    ctx = capi.Context(0)
    plan = capi.Plan(ctx, P.n_qubits, *P.plan_arrays())
    ham = capi.Hamiltonian(ctx, P.n_qubits, *P.ham_arrays())
    order = np.asarray(P.plan.order)

    def fb(X, B):
        X = np.asarray(X).reshape(B, P.n_gen)
        return list(capi.energy_batch(ctx, plan, ham, P.hf, np.ascontiguousarray(X[:, order])))

    opts = ff.OptimizerOptions()
    opts.ftol = 1e-8
    opts.max_evals = 5_000_000
    r = ff.bfgs_minimize(fb, list(P.thetas[0]), opts)
    e_hf = fb(np.zeros(P.n_gen), 1)[0]
    e_cas = capi.lanczos_ground(ctx, ham, P.hf)[0]
    assert r.converged
    assert e_cas - 1e-10 <= r.energy < e_hf


def test_native_vqe_drivers_equal_callback_loops():
    """fragfield::vqe_bfgs / vqe_device build the device objective in C++ (no
    host-language callback inside the loop): at config 2 they follow the
    callback-driven optimizers step for step (same evaluations, same energy and
    amplitudes bit for bit), converge to ftol 1e-8 and stay variational."""
    import paper_2402_17993_b200 as ff

    P = problems.config_problem(2)
    dev = ff.Device(0)
    H = ff.DeviceHamiltonian(dev, P.H)
    plan = ff.DevicePlan(dev, P.plan)
    x0 = list(P.thetas[0])

    def fb(X, B):
        X = np.asarray(X).reshape(B, P.n_gen)
        th = np.ascontiguousarray(X[:, np.asarray(P.plan.order)])
        return list(ff.energy_batch(dev, plan, H, P.hf, th))

    opts = ff.OptimizerOptions()
    opts.ftol = 1e-8
    opts.max_evals = 5_000_000
    a = ff.vqe_bfgs(dev, plan, H, P.hf, x0, opts)
    b = ff.bfgs_minimize(fb, x0, opts)
    assert a.converged and b.converged
    assert (a.n_evals, a.n_iterations, a.energy) == (b.n_evals, b.n_iterations, b.energy)
    assert np.array_equal(np.array(a.x), np.array(b.x))
    e_cas = ff.lanczos_ground(dev, H, P.hf).energy
    assert e_cas - 1e-10 <= a.energy < ff.energy_trotter(dev, [0.0] * P.n_gen, plan, H, P.hf)
    opts.max_evals = 3000
    c = ff.vqe_device(dev, plan, H, P.hf, x0, "powell", opts)
    d = ff.vqe_minimize(lambda x: fb(x, 1)[0], x0, "powell", opts)
    assert (c.n_evals, c.energy) == (d.n_evals, d.energy) and c.energy <= ff.energy_trotter(dev, x0, plan, H, P.hf)
