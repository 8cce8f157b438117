"""Out-of-bounds checks without compute-sanitizer (closed on this pool: runs under it left GPUs
needing a reset). Every operand of a C-ABI call is a view into a larger buffer whose margins
are filled with a NaN canary:

* an out-of-bounds READ that reaches a result turns it non-finite (checked: outputs finite);
* an out-of-bounds WRITE changes the margin (checked: margins still the canary, bit for bit).

Covers the fused operators (fast / tf32 / bf16x3 / fp64, one and two outputs, ragged n and
k off the 32-column / 128-row tiles and the 16-column RHS padding, column-split partials), the
cross operator, the PCG driver with Nystrom and AFN preconditioners, the Woodbury and AFN
applications, the materialised panels and the packed symmetric product."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MARGIN = 4096
CANARY = np.array([0x7FF8DEADBEEF0001], dtype=np.uint64).view(np.float64)[0]  # a NaN payload


@pytest.fixture(scope="module")
def pkg():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_02259_b200 as p

    return p


class Guarded:
    """A (rows, cols) fp64 view with the given strides inside a canary-filled buffer."""

    def __init__(self, rows, cols, col_major=False, fill=None, ld_pad=3):
        import torch

        ld = (rows if col_major else cols) + ld_pad
        span = (cols if col_major else rows) * ld
        self.buf = torch.full((MARGIN + span + MARGIN,), float("nan"), dtype=torch.float64, device="cuda")
        self.buf.view(torch.int64).fill_(int(np.array([CANARY]).view(np.int64)[0]))
        inner = self.buf[MARGIN:MARGIN + span]
        if col_major:
            self.t = inner.view(cols, ld)[:, :rows].T
        else:
            self.t = inner.view(rows, ld)[:, :cols]
        if fill is not None:
            self.t.copy_(fill)
        self.ld = ld
        self.col_major = col_major
        self.span = span

    def strides(self):
        return self.t.stride(0), self.t.stride(1)

    def margins_intact(self):
        import torch

        b = self.buf.view(torch.int64)
        can = int(np.array([CANARY]).view(np.int64)[0])
        ok = bool((b[:MARGIN] == can).all()) and bool((b[MARGIN + self.span:] == can).all())
        # the padding between rows / columns is part of the canary too
        inner = b[MARGIN:MARGIN + self.span]
        if self.col_major:
            pad = inner.view(-1, self.ld)[:, self.t.shape[0]:]
        else:
            pad = inner.view(-1, self.ld)[:, self.t.shape[1]:]
        return ok and bool((pad == can).all())


def _check_product(pkg, kt, n, d, k, precision, nout):
    import torch

    from paper_2503_02259_b200 import _lib

    rng = np.random.default_rng(n * 7 + k)
    x = rng.standard_normal((n, d))
    e = pkg.KernelEngine(pkg.KernelType(kt), x, pkg.Hyperparams(1.1 * np.sqrt(d), 1.2, 0.1), precision=precision)
    b = Guarded(n, k, col_major=True, fill=torch.from_numpy(rng.standard_normal((n, k))).cuda())
    outs = [Guarded(n, k, col_major=False) for _ in range(3)]
    want = [True, nout == 2, nout == 2]
    o_rs, o_cs = outs[0].strides()
    b_rs, b_cs = b.strides()
    _lib.call("kgp_engine_matmul", e.handle, k, b.t.data_ptr(), b_rs, b_cs,
              *(o.t.data_ptr() if w else None for o, w in zip(outs, want)), o_rs, o_cs, None)
    torch.cuda.synchronize()
    for o, w in zip(outs, want):
        assert o.margins_intact(), (kt, n, d, k, precision, "write outside the output")
        if w:
            assert bool(torch.isfinite(o.t).all()), (kt, n, d, k, precision, "non-finite: read outside an input?")
    assert b.margins_intact()
    e.close()


@pytest.mark.parametrize("precision", ["fast", "tf32", "fp64", "bf16x3"])
@pytest.mark.parametrize("n,d,k", [(1, 8, 1), (31, 8, 3), (129, 8, 17), (1000, 8, 33), (4097, 8, 64),
                                   (300, 2, 5), (2049, 4, 33), (777, 3, 130)])
def test_operator_guard_bands(pkg, precision, n, d, k):
    if precision == "bf16x3" and d <= 4:
        pytest.skip("bf16x3 needs d > 4")
    for kt in ("gaussian", "matern52"):
        for nout in (1, 2):
            _check_product(pkg, kt, n, d, k, precision, nout)


def test_solvers_and_preconditioners_guard_bands(pkg):
    """PCG (Nystrom and AFN), the Woodbury / AFN applications and the cross product on guarded
    operands: results finite, margins untouched."""
    import torch

    from paper_2503_02259_b200 import _device, _lib, precond, solver

    rng = np.random.default_rng(5)
    n, d = 1537, 3
    x = rng.uniform(0, 1, (n, d))
    hp = pkg.Hyperparams(0.3, 1.0, 1e-2)
    for prec in ("fp64", "fast"):
        e = pkg.KernelEngine(pkg.KernelType.MATERN32, x, hp, precision=prec)
        for pre in (precond.build(e, 64), precond.build_afn(e, 64, fsai_npt=8)):
            for k in (1, 5, 12):
                b = Guarded(n, k, col_major=True, fill=torch.from_numpy(rng.standard_normal((n, k))).cuda())
                if isinstance(pre, precond.AFNPreconditioner):  # guarded output too (the C entry point)
                    o = Guarded(n, k, col_major=True)
                    b_rs, b_cs = b.strides()
                    o_rs, o_cs = o.strides()
                    _lib.call("kgp_precond_apply_inverse", pre.handle, k, b.t.data_ptr(), b_rs, b_cs,
                              o.t.data_ptr(), o_rs, o_cs, _device.stream_ptr())
                    res = o.t
                else:
                    o, res = None, pre.apply_inverse(b.t)
                torch.cuda.synchronize()
                assert b.margins_intact() and bool(torch.isfinite(res).all()), (prec, k)
                assert o is None or o.margins_intact(), (prec, k)
            y = rng.standard_normal((n, 3))
            rep = solver.pcg_solve(e.matmul, pre.apply_inverse, y, tol=1e-8, max_iter=500)
            assert np.isfinite(rep.solution).all()
        xs = torch.from_numpy(rng.uniform(0, 1, (333, d))).cuda()
        bb = torch.from_numpy(rng.standard_normal((n, 7))).cuda()
        out = e.cross_matmul(xs, bb)
        assert bool(torch.isfinite(out).all())
        e.close()
