"""GPU parity of the reporting calls against the oracle,
through the C ABI: the sequential fine solution, the max-over-time error
(P:651-656), the estimator efficiency (eq. def_efficiency), classical
Parareal with G = 0 and with one coarse backward-Euler step (P:157-158,
P:209-215), and a posteriori stopping (eq. apost_bound)."""
import numpy as np
import pytest

from gpu_util import TAU_1D, gpu_op, gpu_source
from oracle.bounds import a_posteriori, efficiency as oracle_efficiency
from oracle.fine import Op1D, OpPencil, fine, make_op, sequential_reference
from oracle.parareal import parareal as oracle_parareal
from oracle.parareal import parareal_classical as oracle_classical
from oracle.parareal import trajectory_error as oracle_trajectory_error
from oracle.rsvd import rsvd_interval
from workloads import exp2
from workloads import generators as G
from workloads.configs import get

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import torch
    from paper_2508_08873_b200 import build as B
    B.build()
    assert torch.cuda.is_available()


def _u0(cfg):
    import torch
    u0 = np.asarray(G.initial_value(cfg))[None, :]
    return u0, torch.tensor(np.ascontiguousarray(u0.T), dtype=torch.float64, device="cuda")


def _blocks(T, cfg):
    """(n, N+1) tensor -> (N+1, 1, n) oracle blocks."""
    return T.cpu().numpy().T.reshape(cfg.N + 1, 1, cfg.n)


def _coarse(cfg):
    """One backward-Euler step of size Delta T per interval: the GPU operator,
    its source (sampled at t_n = n Delta T), and the oracle's G_n."""
    from paper_2508_08873_b200 import Operator, SourceTerm
    if cfg.problem.startswith("exp2"):
        L, rs, M = exp2.step_matrices(cfg.problem, cfg.n, cfg.T, cfg.N)
        cop = Operator.pencil(*L, cfg.dT, lrowsum=rs, mass=M)
        csrc = exp2.source(cfg.problem, cfg.n, cfg.T, cfg.N)
        oop = OpPencil(L, cfg.dT, 1, rowsum=rs, M=M)
    else:
        rs, cs = G.operator_1d_sums(cfg)
        A = G.operator_1d(cfg)
        cop = Operator.tridiag(*A, cfg.dT, rowsum=rs, colsum=cs)
        sp, tm, am = G.source_1d(cfg)
        csrc = (sp, np.ascontiguousarray(tm[:, cfg.m - 1::cfg.m]), am)   # t_n = n m dt
        oop = Op1D(*A, cfg.dT, 1, rowsum=rs, colsum=cs)
    return cop, SourceTerm.sep1d(*csrc), (lambda n, x: fine(oop, n, x, "affine", csrc))


@pytest.mark.parametrize("name", ["E2", "T1"])
def test_sequential_and_trajectory_error(name):
    import torch
    from paper_2508_08873_b200 import Coarse, parareal, sequential, trajectory_error
    cfg = get(name)
    op = gpu_op(cfg)
    src = gpu_source(cfg)
    u0, u0g = _u0(cfg)
    R = torch.zeros((cfg.n, cfg.N + 1), dtype=torch.float64, device="cuda")
    sequential(op, u0g, src, cfg.N, cfg.m, R)
    op_o = make_op(cfg)
    ref = sequential_reference(op_o, u0, cfg.N, G.source_1d(cfg))
    scale = np.max(np.linalg.norm(ref.reshape(cfg.N + 1, -1), axis=1))
    assert np.max(np.abs(_blocks(R, cfg) - ref)) <= TAU_1D * scale
    # the error of Parareal iterates k = 0, 1 over time
    Gc = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    truncs = [rsvd_interval(op_o, q, cfg.k, cfg.p, cfg.seed_omega) for q in range(1, cfg.N + 1)]
    res = oracle_parareal(op_o, truncs, u0, cfg.N, 1, G.source_1d(cfg))
    for K in (0, 1):
        U = torch.zeros_like(R)
        parareal(Gc, op, u0g, src, K, U, nsrc=1)
        err, ivl = trajectory_error(op, U, R, cfg.N, cfg.m)
        e_or = oracle_trajectory_error(op_o, res.U[K], ref, cfg.N, G.source_1d(cfg))[0]
        assert abs(err[0] - e_or) <= TAU_1D * scale, K
        assert abs(np.max(ivl) - err[0]) == 0.0


@pytest.mark.parametrize("name", ["E2", "T1"])
@pytest.mark.parametrize("coarse", ["zero", "euler"])
def test_classical_parareal_matches_oracle(name, coarse):
    import torch
    from paper_2508_08873_b200 import parareal_classical
    cfg = get(name)
    op = gpu_op(cfg)
    src = gpu_source(cfg)
    u0, u0g = _u0(cfg)
    op_o = make_op(cfg)
    if coarse == "euler":
        cop, csrc, Gfun = _coarse(cfg)
    else:
        cop, csrc, Gfun = None, None, (lambda n, x: np.zeros_like(x))
    K = 4
    U = torch.zeros((cfg.n, cfg.N + 1), dtype=torch.float64, device="cuda")
    upd = parareal_classical(cop, csrc, op, u0g, src, cfg.N, cfg.m, K, U, nsrc=1)
    res = oracle_classical(op_o, Gfun, u0, cfg.N, K, G.source_1d(cfg))
    scale = np.max(np.abs(res.U))
    got = _blocks(U, cfg)
    assert np.max(np.abs(got - res.U[K])) <= TAU_1D * scale
    for k in range(1, K + 1):
        assert np.max(np.abs(upd[k - 1, :, 0] - res.upd[k, :, 0])) <= TAU_1D * scale, k


def test_parareal_tol_stops_where_the_bound_says():
    import torch
    from paper_2508_08873_b200 import Coarse, efficiency, parareal, parareal_tol, sequential, trajectory_error
    cfg = get("T1")
    op = gpu_op(cfg)
    src = gpu_source(cfg)
    u0, u0g = _u0(cfg)
    Gc = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    info = Gc.info()
    d, e = info["delta"], info["eps"]
    K = cfg.K
    U = torch.zeros((cfg.n, cfg.N + 1), dtype=torch.float64, device="cuda")
    upd, _ = parareal(Gc, op, u0g, src, K, U, nsrc=1)
    bound = [max(a_posteriori(d, e, upd[k, :, 0], n) for n in range(1, cfg.N + 1)) for k in range(K)]
    # a tolerance strictly between two consecutive bounds: stop at that iteration
    kk = next(k for k in range(1, K) if bound[k] < bound[k - 1] * 0.5)
    tol = np.sqrt(bound[kk] * bound[kk - 1])
    U2 = torch.zeros_like(U)
    kd, upd2, _ = parareal_tol(Gc, op, u0g, src, K, tol, U2, nsrc=1)
    assert kd == kk + 1
    U3 = torch.zeros_like(U)
    parareal(Gc, op, u0g, src, kd, U3, nsrc=1)
    assert torch.equal(U2, U3)
    assert np.array_equal(upd2, upd[:kd])
    # efficiency of the estimator (eq. def_efficiency) vs the oracle formula
    R = torch.zeros_like(U)
    sequential(op, u0g, src, cfg.N, cfg.m, R)
    te = []
    for k in range(0, 3):
        Uk = torch.zeros_like(U)
        parareal(Gc, op, u0g, src, k, Uk, nsrc=1)
        te.append(trajectory_error(op, Uk, R, cfg.N, cfg.m)[0][0])
    eta = efficiency(d, e, upd[:2, :, 0], np.array(te))
    for k in (1, 2):
        ref = oracle_efficiency(d, e, upd[k - 1, :, 0], te[k], cfg.N)
        assert abs(eta[k - 1] - ref) <= 1e-14 * abs(ref)
