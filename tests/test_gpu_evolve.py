"""EvolveGCN-O weight-evolution kernels (csrc/evolve.cu) against the oracle's
fp64 recurrence (oracle/dgnn.py evolve_forward / evolve_backward), for every
kernel family: the register-resident 2-CTA cluster kernels (F_l = 128, 1/2/4
columns per cluster, ragged column counts) and the L2-streamed kernels."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

VARIANTS = ["rr2", "rr1", "rr4", "0"]


def _problem(Fl, Hl, T, seed):
    rng = np.random.default_rng(seed)
    W0 = rng.normal(0, 0.5, (Fl, Hl))
    Sr, Sz, Pc, Qc = (rng.normal(0, 1.0 / np.sqrt(Fl), (Fl, Fl)) for _ in range(4))
    Br, Bz, Bc = (rng.normal(0, 0.1, (Fl, Hl)) for _ in range(3))
    dWd = rng.normal(0, 1.0, (T, Fl, Hl))
    return W0, Sr, Sz, Pc, Qc, Br, Bz, Bc, dWd


def _run(variant, Fl, Hl, T, prob):
    from paper_2309_03523_b200 import ops
    W0, Sr, Sz, Pc, Qc, Br, Bz, Bc, dWd = prob
    dev = torch.device("cuda:0")
    f = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32, device=dev)
    Wstack = torch.zeros(((T + 1) * Fl, Hl), dtype=torch.float32, device=dev)
    sv = [torch.zeros((Fl, T * Hl), dtype=torch.float32, device=dev) for _ in range(5)]
    da = [torch.zeros((Fl, T * Hl), dtype=torch.float32, device=dev) for _ in range(3)]
    dB = [torch.zeros((Fl, Hl), dtype=torch.float32, device=dev) for _ in range(3)]
    dW0 = torch.zeros((Fl, Hl), dtype=torch.float32, device=dev)
    old = os.environ.pop("DGC_EVOLVE_CL", None)
    if variant is not None:
        os.environ["DGC_EVOLVE_CL"] = variant
    try:
        ops.evolve_fwd(Fl, Hl, T, f(W0), f(Sr), f(Sz), f(Pc), f(Qc), f(Br), f(Bz), f(Bc), Wstack, sv)
        ops.evolve_bwd(Fl, Hl, T, f(Sr), f(Sz), f(Pc), f(Qc), sv, f(dWd.reshape(T * Fl, Hl)),
                       dW0, da, dB)
        torch.cuda.synchronize()
    finally:
        if old is None:
            os.environ.pop("DGC_EVOLVE_CL", None)
        else:
            os.environ["DGC_EVOLVE_CL"] = old
    return (Wstack.cpu().numpy().astype(np.float64), [x.cpu().numpy().astype(np.float64) for x in sv],
            dW0.cpu().numpy().astype(np.float64), [x.cpu().numpy().astype(np.float64) for x in da],
            [x.cpu().numpy().astype(np.float64) for x in dB])


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("Fl,Hl,T", [(128, 128, 12), (128, 37, 9), (32, 20, 7)])
def test_evolve_kernels_match_oracle(variant, Fl, Hl, T):
    from oracle.dgnn import evolve_backward, evolve_forward
    prob = _problem(Fl, Hl, T, Fl + Hl + T)
    W0, Sr, Sz, Pc, Qc, Br, Bz, Bc, dWd = prob
    Ws, saves = evolve_forward(W0, Sr, Sz, Pc, Qc, Br, Bz, Bc, T)
    ref = evolve_backward(Sr, Sz, Pc, Qc, saves, list(dWd))
    Wstack, sv, dW0, da, dB = _run(variant, Fl, Hl, T, prob)
    tol = 2e-5
    assert _rel(Wstack.reshape(T + 1, Fl, Hl), np.stack(Ws)) <= tol
    # saves [Fl][T][Hl]: r z c w rw
    for t in range(T):
        w, r, z, c = saves[t]
        for got, want in ((sv[0], r), (sv[1], z), (sv[2], c), (sv[3], w), (sv[4], r * w)):
            assert _rel(got[:, t * Hl:(t + 1) * Hl], want) <= tol
    carry, g_Sr, g_Sz, g_Pc, g_Qc, g_Br, g_Bz, g_Bc = ref
    assert _rel(dW0, carry) <= 1e-4
    assert _rel(dB[0], g_Br) <= 1e-4 and _rel(dB[1], g_Bz) <= 1e-4 and _rel(dB[2], g_Bc) <= 1e-4
    # gate-matrix gradients as the trainer forms them: da (Fl x T*Hl) @ saved operand^T
    assert _rel(da[0] @ sv[3].T, g_Sr) <= 1e-4
    assert _rel(da[1] @ sv[3].T, g_Sz) <= 1e-4
    assert _rel(da[2] @ sv[3].T, g_Pc) <= 1e-4
    assert _rel(da[2] @ sv[4].T, g_Qc) <= 1e-4


def test_evolve_cluster_kernel_is_default_at_128():
    """With no override the C3/C5 shape (F_l = 128) runs the register-resident
    2-column cluster kernels: bitwise the rr2 results, not the L2 kernels'."""
    Fl, Hl, T = 128, 128, 4
    prob = _problem(Fl, Hl, T, 1)
    rr2, l2, default = (_run(v, Fl, Hl, T, prob) for v in ("rr2", "0", None))
    assert np.array_equal(default[0], rr2[0]) and np.array_equal(default[2], rr2[2])
    assert not np.array_equal(default[2], l2[2])  # different summation order
