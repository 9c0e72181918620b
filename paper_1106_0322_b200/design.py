"""Device-resident design matrix (the layouts libspa_b200 reads).

Built once per (dataset, intercept) from the host arrays the reference uses
(reference smc.py:106-123 `make_design`: optional leading unpenalised column
of ones).  Two representations:

* coded (the genotype case): every column takes at most 3 equally spaced
  values, x = alpha*g + gamma with g in {0,1,2} (standardised allele counts,
  reference data.py:131-140, are exactly this).  The tensor-core operand is
  the byte planes [G | 64 G] for the int8 likelihood kernel and the MwG
  kernel reads 2-bit codes from two bit planes.
* general: arbitrary float columns; the tensor-core operand is the fp16
  hi/lo split [Xhi | Xlo] and the MwG kernel reads float32 columns.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from ._lib import SpaDesign

K_ALIGN = 64


def _round_up(x: int, m: int) -> int:
    return -(-x // m) * m


def mwg_words(n: int) -> int:
    """32-subject words per column so that the MwG kernel's thread layout
    (csrc/mwg.cu: S subjects per thread, >= 32 threads) is fully covered."""
    S = 8 if n <= 256 else (16 if n <= 512 else 32)
    nthr = max(32, _round_up(-(-n // S), 32))
    return -(-(nthr * S) // 32)


def _code_column(x: np.ndarray):
    """Return (codes, alpha, gamma, levels) if x = alpha*g + gamma with
    g in {0,1,2} (at most 3 equally spaced distinct values), else None."""
    u = np.unique(x)
    if u.size == 1:
        return np.zeros(x.size, np.uint8), 0.0, float(u[0]), np.array([u[0], 0.0, 0.0])
    if u.size > 3:
        return None
    step = float(u[1] - u[0])
    if u.size == 3 and abs((u[2] - u[1]) - step) > 1e-9 * max(1.0, abs(step)):
        return None
    g = np.rint((x - u[0]) / step)
    if np.max(np.abs(u[0] + step * g - x)) > 1e-12 * max(1.0, float(np.max(np.abs(x)))):
        return None
    lev = np.zeros(3)
    lev[: u.size] = u
    return g.astype(np.uint8), step, float(u[0]), lev


def _code_columns(X: np.ndarray, dev) -> list:
    """_code_column for every column at once, on the device (float64; the
    per-column np.unique sorts took ~40 ms at n=5000, p=500).  Division and
    rint are exactly rounded, so the codes, steps and levels are identical
    to the host function's."""
    n, q = X.shape
    XT = torch.from_numpy(np.ascontiguousarray(X.T)).to(dev)
    mn, mx = XT.min(dim=1).values, XT.max(dim=1).values
    inf = torch.tensor(float("inf"), dtype=XT.dtype, device=dev)
    u1 = torch.where(XT > mn[:, None], XT, inf).min(dim=1).values  # second smallest distinct value
    const = mn == mx
    in_set = ((XT == mn[:, None]) | (XT == u1[:, None]) | (XT == mx[:, None])).all(dim=1) | const
    step = torch.where(const, torch.ones_like(mn), u1 - mn)
    three = (u1 < mx) & ~const
    spaced = ~three | ((mx - u1 - step).abs() <= 1e-9 * torch.clamp(step.abs(), min=1.0))
    G = torch.round((XT - mn[:, None]) / step[:, None])  # round half to even, as np.rint
    err = (mn[:, None] + step[:, None] * G - XT).abs().max(dim=1).values
    exact = err <= 1e-12 * torch.clamp(XT.abs().max(dim=1).values, min=1.0)
    ok = (in_set & (const | (spaced & exact))).cpu().numpy()
    codes = torch.where(const[:, None], torch.zeros_like(G), G).to(torch.uint8).cpu().numpy()
    mn, u1, mx, step = (v.cpu().numpy() for v in (mn, u1, mx, step))
    const, three = const.cpu().numpy(), three.cpu().numpy()
    out = [None] * q
    for j in np.flatnonzero(ok):
        if const[j]:
            out[j] = (codes[j], 0.0, float(mn[j]), np.array([mn[j], 0.0, 0.0]))
        else:
            lev = np.zeros(3)
            lev[: 3 if three[j] else 2] = (mn[j], u1[j], mx[j]) if three[j] else (mn[j], u1[j])
            out[j] = (codes[j], float(step[j]), float(mn[j]), lev)
    return out


@dataclass
class DeviceDesign:
    """Owns the device tensors behind one `spa_design` struct."""

    n: int
    q: int
    coded: bool
    kp: int
    penalized: np.ndarray
    tensors: dict
    struct: SpaDesign

    @property
    def ptr(self):
        return self.struct

    @classmethod
    def build(cls, X, y, intercept: bool = False, device=None) -> "DeviceDesign":
        X = np.asarray(X, dtype=np.float64)
        y = np.asarray(y, dtype=np.float64)
        if intercept:
            X = np.column_stack([np.ones(X.shape[0]), X])
        n, q = X.shape
        pen = np.ones(q, dtype=np.uint8)
        if intercept:
            pen[0] = 0
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        coded_cols = _code_columns(X, dev)
        coded = all(c is not None for c in coded_cols)
        n_words = mwg_words(n)
        npad = n_words * 32
        sy = X.T @ y
        t = {}
        if coded:
            codes = np.stack([c[0] for c in coded_cols])  # [q][n]
            alpha = np.array([c[1] for c in coded_cols])
            gamma = np.array([c[2] for c in coded_cols])
            lev = np.zeros((q, 4), np.float32)
            lev[:, :3] = np.stack([c[3] for c in coded_cols])
            b1 = np.zeros((q, npad), bool)
            b2 = np.zeros((q, npad), bool)
            b1[:, :n] = codes == 1
            b2[:, :n] = codes == 2
            b1[:, n:] = True  # padding subjects carry code (1,1)
            b2[:, n:] = True
            p1 = np.packbits(b1, axis=1, bitorder="little").view("<u4")
            p2 = np.packbits(b2, axis=1, bitorder="little").view("<u4")
            planes = np.stack([p1, p2], axis=-1).astype(np.uint32)  # [q][n_words][2]
            # MwG codes: 16 subjects per word, subject s in bits 2s..2s+1 (3 = padding)
            cc = np.full((q, npad), 3, np.uint32)
            cc[:, :n] = codes
            words = (cc.reshape(q, npad // 16, 16) << (2 * np.arange(16, dtype=np.uint32))).sum(axis=2, dtype=np.uint64)
            t["codes"] = torch.from_numpy(words.astype(np.uint32).view(np.int32)).to(dev)
            # int8 K1 operand (csrc/tc_k1_i8.cuh): two byte planes [G | 64 G]
            kp = _round_up(q, K_ALIGN)
            G = np.zeros((n, 2 * kp), np.uint8)
            G[:, :q] = codes.T
            G[:, kp:kp + q] = 64 * codes.T
            t["planes"] = torch.from_numpy(planes.view(np.int32).copy()).to(dev)
            t["xlev"] = torch.from_numpy(lev).to(dev)
            t["alpha"] = torch.from_numpy(alpha).to(dev)
            t["gamma"] = torch.from_numpy(gamma).to(dev)
            t["gemm_b"] = torch.from_numpy(G).to(dev).contiguous()
            terms = 1
        else:
            kp = _round_up(q, K_ALIGN)
            xc = np.zeros((q, npad), np.float32)
            xc[:, :n] = X.T
            t["xcols"] = torch.from_numpy(xc).to(dev)
            # fp16 hi/lo operand of X scaled per column by a power of two
            # (max |X_j| / 2^s_j in [2, 8)); the pack multiplies beta_j by
            # alpha_j = 2^s_j, so the product is unchanged and both fp16
            # terms stay in their normal range
            mx = np.max(np.abs(X), axis=0) if n else np.zeros(q)
            sh = np.where(mx > 0, np.round(np.log2(np.where(mx > 0, mx, 1.0))) - 2, 0).astype(np.int64)
            scale = np.ldexp(1.0, sh)
            Xf = torch.zeros((n, kp), dtype=torch.float64)
            Xf[:, :q] = torch.from_numpy(X / scale)
            hi = Xf.to(torch.float16)
            lo = (Xf - hi.to(torch.float64)).to(torch.float16)
            t["gemm_b"] = torch.cat([hi, lo], dim=1).contiguous().to(dev)
            t["xlev"] = torch.zeros((q, 4), dtype=torch.float32, device=dev)
            t["alpha"] = torch.from_numpy(scale).to(dev)  # K1 column scale (general designs)
            t["gamma"] = torch.zeros(q, dtype=torch.float64, device=dev)
            terms = 2
        t["sy"] = torch.from_numpy(sy).to(dev)
        t["sx"] = torch.from_numpy(X.sum(axis=0)).to(dev)  # X^T 1: the linear half of the coded K1 softplus
        t["penalized"] = torch.from_numpy(pen).to(dev)
        s = SpaDesign()
        s.n, s.q, s.coded, s.n_words = n, q, int(coded), n_words
        s.planes = t["planes"].data_ptr() if coded else None
        s.xcols = None if coded else t["xcols"].data_ptr()
        s.xlev = t["xlev"].data_ptr()
        s.sy = t["sy"].data_ptr()
        s.sx = t["sx"].data_ptr()
        s.alpha = t["alpha"].data_ptr()
        s.gamma = t["gamma"].data_ptr()
        s.penalized = t["penalized"].data_ptr()
        s.gemm_b = t["gemm_b"].data_ptr()
        s.kp, s.terms = kp, terms
        s.codes = t["codes"].data_ptr() if coded else None
        return cls(n, q, coded, kp, pen.astype(bool), t, s)
