"""Out-of-bounds and uninitialised-read guards for the library's entry points.

compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing
a reset), so the memcheck / initcheck questions are asked directly:

* every output buffer is followed by a canary region that must be untouched
  after the call (an out-of-bounds store past any output fails);
* every workspace and every buffer the callee fully overwrites is poisoned
  (NaN / random bytes) first -- a kernel reading uninitialised scratch would
  change the result, which must equal the clean run bit for bit.

Shapes are ragged on purpose (particle counts that are not multiples of the
128-row tiles, q not a multiple of 4 / 16) so tail tiles and row ends are hit.
"""

import ctypes
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1106_0322_b200 import _lib  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402
from paper_1106_0322_b200.design import DeviceDesign  # noqa: E402
from paper_1106_0322_b200.smc import ParticleSystem, _p, _stream  # noqa: E402

CANARY = 0x5A
PAD = 4096  # bytes of canary after every output


class Guarded:
    """A tensor view with PAD canary bytes behind it in the same allocation."""

    def __init__(self, shape, dtype, fill=None):
        n = int(np.prod(shape)) * torch.tensor([], dtype=dtype).element_size()
        self.raw = torch.full((n + PAD,), CANARY, dtype=torch.uint8, device="cuda")
        self.t = self.raw[:n].view(dtype).view(shape)
        if fill is not None:
            self.t.fill_(fill)

    def intact(self):
        return bool((self.raw[-PAD:] == CANARY).all())


def poisoned(nbytes):
    g = torch.Generator(device="cuda")
    g.manual_seed(nbytes)
    return torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device="cuda", generator=g)


def _system(name, N, seed=0):
    data, _ = simulate_dataset(named_spec(name))
    d = DeviceDesign.build(data.X, data.y, False)
    s = ParticleSystem(d, N, 1.0, False)
    rng = np.random.default_rng(seed)
    s.load_betas(rng.normal(0.0, 0.1, size=(N, d.q)))
    return data, d, s


@pytest.mark.parametrize("name,N", [("c1", 1000), ("c2", 333), ("c3", 1037)])
def test_loglik_guards(name, N):
    data, d, s = _system(name, N)
    nws = _lib.load().spa_loglik_workspace_bytes(N, d.n)
    a_bytes = _lib.load().spa_k1_operand_bytes(ctypes.byref(d.struct), N)
    outs = []
    for poison in (False, True):
        A = Guarded((a_bytes,), torch.uint8, 0xFF if poison else 0)
        yl = Guarded((N,), torch.float64, float("nan") if poison else 0.0)
        out = Guarded((N,), torch.float64, float("nan"))
        ws = poisoned(nws) if poison else torch.zeros(nws, dtype=torch.uint8, device="cuda")
        _lib.call("spa_loglik_rows", ctypes.byref(d.struct), _p(s.beta), N, s.ldb, _p(A.t), _p(yl.t), _p(out.t),
                  _p(ws), nws, _stream())
        torch.cuda.synchronize()
        assert A.intact() and yl.intact() and out.intact()
        assert bool(torch.isfinite(out.t).all())
        outs.append(out.t.clone())
    assert torch.equal(outs[0], outs[1])


def test_rw_move_guards():
    """Propose (L z GEMM + pack), K1 and accept with a ragged N at C2."""
    from paper_1106_0322_b200.smc import _round_up, _rw_factor

    data, d, s = _system("c2", 1001, seed=3)
    s.log_weights = np.full(s.N, -math.log(s.N))
    _rw_factor(s, 2.38)
    rw, ws = s.rw_workspace(), s.ll_workspace()
    q, kq, N = s.q, _round_up(s.q, 64), s.N
    zb = s.z_buffers(1)[0]
    _lib.call("spa_rw_normals", N, q, 3, 5, 0, 1, _p(zb), _stream())
    res = []
    for poison in (False, True):
        eps = Guarded((N, s.ldb), torch.bfloat16, float("nan") if poison else 0.0)
        eps.t[:, q:] = 0  # the padding columns are the caller's (zero) contract
        A = Guarded((_lib.load().spa_k1_operand_bytes(ctypes.byref(d.struct), N),), torch.uint8,
                    0xFF if poison else 0)
        yl = Guarded((N,), torch.float64, float("nan"))
        lp = Guarded((N,), torch.float64, float("nan"))
        sp = Guarded((N,), torch.float64, float("nan"))
        nws = ws["ws"].numel()
        kws = poisoned(nws) if poison else torch.zeros(nws, dtype=torch.uint8, device="cuda")
        _lib.call("spa_rw_propose", ctypes.byref(d.struct), _p(s.beta), N, s.ldb, s.factor_operand(), 3, 5, 0, 1,
                  _p(zb), _p(eps.t), _p(A.t), _p(yl.t), 1.0, 0.9, _p(lp.t), _stream())
        _lib.call("spa_loglik_softplus", ctypes.byref(d.struct), _p(A.t), N, _p(sp.t), _p(kws), nws, _stream())
        beta = Guarded((N, s.ldb), torch.float32)
        beta.t.copy_(s.beta)
        ll = Guarded((N,), torch.float64)
        ll.t.copy_(s.ll)
        lpc = Guarded((N,), torch.float64)
        lpc.t.fill_(-1.0)
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        _lib.call("spa_rw_accept", _p(beta.t), s.ldb, _p(eps.t), q, N, _p(yl.t), _p(sp.t), _p(lp.t), _p(ll.t),
                  _p(lpc.t), 3, 5, 0, 1, _p(cnt), _stream())
        torch.cuda.synchronize()
        for g in (eps, A, yl, lp, sp, beta, ll, lpc):
            assert g.intact()
        assert bool(torch.isfinite(sp.t).all()) and bool(torch.isfinite(yl.t).all())
        res.append((eps.t[:, :q].clone(), sp.t.clone(), beta.t[:, :q].clone(), int(cnt.item())))
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])
    assert torch.equal(res[0][2], res[1][2]) and res[0][3] == res[1][3]


@pytest.mark.parametrize("N", [7, 2049, 65539])
def test_resample_guards(N):
    q, ldb = 13, 16
    rng = np.random.default_rng(N)
    w = torch.from_numpy(rng.dirichlet(np.full(N, 0.5))).cuda()
    src = torch.randn((N, ldb), device="cuda")
    outs = []
    nws = _lib.load().spa_resample_workspace_bytes(N)
    for poison in (False, True):
        ws = poisoned(nws) if poison else torch.zeros(nws, dtype=torch.uint8, device="cuda")
        beta = Guarded((N, ldb), torch.float32)
        beta.t.copy_(src)
        alt = Guarded((N, ldb), torch.float32, float("nan") if poison else 0.0)
        ll, lp = Guarded((N,), torch.float64, 1.0), Guarded((N,), torch.float64, 2.0)
        lla, lpa = Guarded((N,), torch.float64, float("nan")), Guarded((N,), torch.float64, float("nan"))
        logw = Guarded((N,), torch.float64, 0.0)
        anc = Guarded((N,), torch.int64, -1)
        gate = torch.ones(1, dtype=torch.float64, device="cuda")
        _lib.call("spa_resample_gated", _p(gate), _p(w), N, 0.41 / N, _p(beta.t), _p(alt.t), ldb, q, _p(ll.t),
                  _p(lla.t), _p(lp.t), _p(lpa.t), _p(logw.t), _p(anc.t), _p(ws), nws, _stream())
        torch.cuda.synchronize()
        for g in (beta, alt, ll, lp, lla, lpa, logw, anc):
            assert g.intact()
        outs.append((anc.t.clone(), beta.t[:, :q].clone()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def test_mwg_and_summary_guards():
    data, d, s = _system("c1", 333, seed=5)
    beta = Guarded((s.N, s.ldb), torch.float32)
    beta.t.copy_(s.beta)
    ll, lp = Guarded((s.N,), torch.float64, float("nan")), Guarded((s.N,), torch.float64, float("nan"))
    cnt = Guarded((1,), torch.int64, 0)
    _lib.call("spa_mwg_move", ctypes.byref(d.struct), _p(beta.t), s.N, s.ldb, 1.0, 0.5, 0.5, 2, 7, 1, 3, 0, 0,
              _p(ll.t), _p(lp.t), _p(cnt.t), 0, _stream())
    torch.cuda.synchronize()
    assert beta.intact() and ll.intact() and lp.intact() and cnt.intact()
    assert bool(torch.isfinite(ll.t).all()) and bool(torch.isfinite(lp.t).all())
    from paper_1106_0322_b200.smc import _weighted_marginals

    w = torch.full((s.N,), 1.0 / s.N, dtype=torch.float64, device="cuda")
    out = _weighted_marginals(beta.t, s.N, s.ldb, s.q, w, (0.05, 0.5, 0.95), (0.1,))
    torch.cuda.synchronize()
    assert beta.intact()
    assert all(bool(torch.isfinite(v).all()) for v in out.values())
