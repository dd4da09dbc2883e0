"""Host-buffer path of pq_phi_0p with PINNED output buffers: phi_0 is copied out on the side stream
while the squaring runs (capi.cpp run_phiquadmv).  The results must equal the device-resident path
bitwise and be complete when the call returns (no later synchronisation by the caller)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("memory", ["pinned", "pageable"])
@pytest.mark.parametrize("cfg,n", [(2, 16), (2, 64), (2, 128), (3, 64), (5, 64)])
def test_pinned_host_outputs_equal_device_outputs(pq, cfg, n, memory):
    """(2, 64), (2, 128), (3, 64), (5, 64): the two-group squaring with the run-ahead lower half
    (uneven halves at p = 3); (2, 16): below the split threshold.  Pageable buffers go through the
    engine's pinned bounce, with the early copies drained while the call runs (capi.cpp)."""
    import torch
    from paper_2211_00696_b200.workloads import config
    w = config(cfg, n=n)
    a = pq.KroneckerSum(w.factors)
    req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
    b = w.rhs(5)
    ctx = pq.Context(0)
    d, sh, fac = a._abi()
    rc = req._c()
    info = pq._lib.PhiInfoC()
    b_dev = torch.from_numpy(b).cuda()
    o0_dev = torch.empty((1, w.N), dtype=torch.float64, device="cuda")
    o_dev = torch.empty((1, w.p, w.N), dtype=torch.float64, device="cuda")
    pq._lib.check(pq._lib.lib.pq_phi_0p(ctx.handle, d, sh, fac, 1, C.c_void_p(b_dev.data_ptr()), C.byref(rc),
                                        C.c_void_p(o0_dev.data_ptr()), C.c_void_p(o_dev.data_ptr()), C.byref(info),
                                        pq._lib.PQ_DEVICE))
    torch.cuda.synchronize()
    b_pin = torch.from_numpy(b.copy()).pin_memory()
    o0_pin = torch.full((1, w.N), np.nan, dtype=torch.float64).pin_memory()
    o_pin = torch.full((1, w.p, w.N), np.nan, dtype=torch.float64).pin_memory()
    # three calls on the same context (warm workspaces and helper streams), the third into fresh
    # output buffers
    def fresh(shape):
        t = torch.full(shape, np.nan, dtype=torch.float64)
        return t.pin_memory() if memory == "pinned" else t

    if memory == "pageable":
        b_pin = torch.from_numpy(b.copy())
    for k in range(3):
        if k == 2 or memory == "pageable":
            o0_pin = fresh((1, w.N))
            o_pin = fresh((1, w.p, w.N))
        else:
            o0_pin.fill_(np.nan)
            o_pin.fill_(np.nan)
        pq._lib.check(pq._lib.lib.pq_phi_0p(ctx.handle, d, sh, fac, 1, C.c_void_p(b_pin.data_ptr()), C.byref(rc),
                                            C.c_void_p(o0_pin.data_ptr()), C.c_void_p(o_pin.data_ptr()),
                                            C.byref(info), pq._lib.PQ_HOST))
        # read immediately: the call must have completed every copy it issued
        assert np.array_equal(o0_pin.numpy(), o0_dev.cpu().numpy()), k
        assert np.array_equal(o_pin.numpy(), o_dev.cpu().numpy()), k
    ctx.close()


def test_two_host_callers_concurrently_match_sequential(pq):
    """bench.py's end-to-end leg runs two host threads, each with its own context, stream and
    pinned buffers, calling pq_phi_0p at once (the reference API is re-entrant).  Every result
    must equal the same call made alone, bitwise, across several overlapped rounds."""
    import threading
    import torch
    from paper_2211_00696_b200.workloads import config
    w = config(2, n=64)
    a = pq.KroneckerSum(w.factors)
    req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
    d, sh, fac = a._abi()
    rc = req._c()
    rhs = [w.rhs(10 + k) for k in range(2)]

    def make():
        ctx = pq.Context(0)
        st = torch.cuda.Stream()
        ctx.set_stream(st.cuda_stream)
        return ctx, st

    def call(ctx, b, o0, o):
        info = pq._lib.PhiInfoC()
        pq._lib.check(pq._lib.lib.pq_phi_0p(ctx.handle, d, sh, fac, 1, C.c_void_p(b.data_ptr()), C.byref(rc),
                                            C.c_void_p(o0.data_ptr()), C.c_void_p(o.data_ptr()), C.byref(info),
                                            pq._lib.PQ_HOST))

    callers = [make() for _ in range(2)]
    bufs = [(torch.from_numpy(rhs[k].copy()).pin_memory(), torch.empty((1, w.N), dtype=torch.float64).pin_memory(),
             torch.empty((1, w.p, w.N), dtype=torch.float64).pin_memory()) for k in range(2)]
    want = []
    for k in range(2):
        call(callers[k][0], *bufs[k])
        want.append((bufs[k][1].numpy().copy(), bufs[k][2].numpy().copy()))
    errors = []

    def worker(k):
        try:
            for _ in range(3):
                bufs[k][1].fill_(float("nan"))
                bufs[k][2].fill_(float("nan"))
                call(callers[k][0], *bufs[k])
                if not (np.array_equal(bufs[k][1].numpy(), want[k][0]) and np.array_equal(bufs[k][2].numpy(), want[k][1])):
                    errors.append(f"caller {k}: result differs from the sequential call")
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))

    ths = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors, errors
    for ctx, _ in callers:
        ctx.close()


@pytest.mark.parametrize("n", [32, 64, 104])
@pytest.mark.parametrize("space", ["host", "device"])
def test_phiquadmv_cols_equals_contiguous(pq, space, n):
    """pq_phiquadmv_cols (the drop-in headers' entry: each RHS and each result column at its own
    address) returns bitwise what pq_phiquadmv returns in one contiguous buffer, nb = 2.  n = 32
    (262 k doubles of results) takes the direct-copy branch, n = 64 (2 M doubles >= the 8 MB bounce
    threshold) the pinned bounce with the early drain and the final scatter (capi.cpp); n = 104
    (2 x 1.1 M doubles of right-hand sides) also the gathered input bounce (gather_cols), and the
    contiguous call the pageable input bounce (stage_in)."""
    import torch
    from paper_2211_00696_b200.workloads import config
    w = config(2, n=n)
    a = pq.KroneckerSum(w.factors)
    req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
    ctx = pq.Context(0)
    d, sh, fac = a._abi()
    rc = req._c()
    nb, N, p = 2, w.N, w.p
    bs = np.stack([w.rhs(20), w.rhs(21)])
    want = np.empty((nb, p, N))
    info = pq._lib.PhiInfoC()
    pq._lib.check(pq._lib.lib.pq_phiquadmv(ctx.handle, d, sh, fac, nb, C.c_void_p(bs.ctypes.data), C.byref(rc),
                                           C.c_void_p(want.ctypes.data), C.byref(info), pq._lib.PQ_HOST))
    if space == "host":
        b_sep = [np.ascontiguousarray(bs[m]) for m in range(nb)]
        cols = [np.full(N, np.nan) for _ in range(nb * p)]
        bptr = [x.ctypes.data for x in b_sep]
        cptr = [x.ctypes.data for x in cols]
        sp = pq._lib.PQ_HOST
    else:
        b_sep = [torch.from_numpy(bs[m].copy()).cuda() for m in range(nb)]
        cols = [torch.full((N,), float("nan"), dtype=torch.float64, device="cuda") for _ in range(nb * p)]
        bptr = [x.data_ptr() for x in b_sep]
        cptr = [x.data_ptr() for x in cols]
        sp = pq._lib.PQ_DEVICE
    barr = (C.c_void_p * nb)(*bptr)
    carr = (C.c_void_p * (nb * p))(*cptr)
    info2 = pq._lib.PhiInfoC()
    pq._lib.check(pq._lib.lib.pq_phiquadmv_cols(ctx.handle, d, sh, fac, nb, barr, C.byref(rc), carr, C.byref(info2), sp))
    torch.cuda.synchronize()
    got = np.stack([np.asarray(c.cpu() if space == "device" else c) for c in cols]).reshape(nb, p, N)
    assert np.array_equal(got, want)
    assert (info2.l, info2.n, info2.points) == (info.l, info.n, info.points)
    ctx.close()


@pytest.mark.parametrize("n", [32, 64])
@pytest.mark.parametrize("kind", [0, 1])
def test_phi_with_plan_cols_equals_contiguous(pq, kind, n):
    """pq_phi_with_plan_cols (drop-in phi_with_plan / PhiEngine::apply) returns bitwise what
    pq_phi_with_plan returns contiguously; nb = 2 pageable host vectors, both rules; n = 64 crosses
    the pinned-bounce threshold (one D2H into the bounce, host threads fill the columns)."""
    from paper_2211_00696_b200.workloads import config
    w = config(2, n=n)
    a = pq.KroneckerSum(w.factors)
    ctx = pq.Context(0)
    d, sh, fac = a._abi()
    nb, N, p, l, n = 2, w.N, w.p, 3, 8
    mode = pq._lib.PQ_GAUSS_LEGENDRE if kind == 0 else pq._lib.PQ_CLENSHAW_CURTIS
    bs = np.stack([w.rhs(30), w.rhs(31)])
    want = np.empty((nb, p, N))
    pts = C.c_int(0)
    pq._lib.check(pq._lib.lib.pq_phi_with_plan(ctx.handle, d, sh, fac, nb, C.c_void_p(bs.ctypes.data), p, l, n, mode,
                                               w.eps, C.c_void_p(want.ctypes.data), C.byref(pts), pq._lib.PQ_HOST))
    b_sep = [np.ascontiguousarray(bs[m]) for m in range(nb)]
    cols = [np.full(N, np.nan) for _ in range(nb * p)]
    barr = (C.c_void_p * nb)(*[x.ctypes.data for x in b_sep])
    carr = (C.c_void_p * (nb * p))(*[x.ctypes.data for x in cols])
    pts2 = C.c_int(0)
    pq._lib.check(pq._lib.lib.pq_phi_with_plan_cols(ctx.handle, d, sh, fac, nb, barr, p, l, n, mode, w.eps, carr,
                                                    C.byref(pts2), pq._lib.PQ_HOST))
    assert np.array_equal(np.stack(cols).reshape(nb, p, N), want)
    assert pts2.value == pts.value
    ctx.close()


@pytest.mark.parametrize("n", [16, 64])
def test_fixed_adaptive_squaring_cols_equal_contiguous(pq, n):
    """pq_phi_fixed_cols / pq_phi_adaptive_cols / pq_squaring_step_cols (the drop-in headers'
    phi_fixed_multi, phi_adaptive_multi and squaring_step on the caller's vectors) return bitwise
    what the contiguous entry points return; n = 64 crosses the pinned-bounce threshold."""
    from paper_2211_00696_b200.workloads import config
    w = config(2, n=n)
    a = pq.KroneckerSum(w.factors)
    ctx = pq.Context(0)
    d, sh, fac = a._abi()
    nb, N, p = 2, w.N, w.p
    bs = np.stack([w.rhs(40), w.rhs(41)])
    b_sep = [np.ascontiguousarray(bs[m]) for m in range(nb)]
    barr = (C.c_void_p * nb)(*[x.ctypes.data for x in b_sep])
    H = pq._lib.PQ_HOST
    rule = pq.cached_rule(pq.QuadKind.gauss_legendre, 9)
    x, wt = np.ascontiguousarray(rule.nodes), np.ascontiguousarray(rule.weights)
    want = np.empty((nb, p, N))
    pq._lib.check(pq._lib.lib.pq_phi_fixed(ctx.handle, d, sh, fac, nb, C.c_void_p(bs.ctypes.data), p, 9,
                                           x.ctypes.data_as(pq._lib.dp), wt.ctypes.data_as(pq._lib.dp),
                                           C.c_void_p(want.ctypes.data), H))
    cols = [np.full(N, np.nan) for _ in range(nb * p)]
    carr = (C.c_void_p * (nb * p))(*[c.ctypes.data for c in cols])
    pq._lib.check(pq._lib.lib.pq_phi_fixed_cols(ctx.handle, d, sh, fac, nb, barr, p, 9, x.ctypes.data_as(pq._lib.dp),
                                                wt.ctypes.data_as(pq._lib.dp), carr, H))
    assert np.array_equal(np.stack(cols).reshape(nb, p, N), want)
    want = np.empty((nb, p, N))
    pts, pts2 = C.c_int(), C.c_int()
    pq._lib.check(pq._lib.lib.pq_phi_adaptive(ctx.handle, d, sh, fac, nb, C.c_void_p(bs.ctypes.data), p, 1e-10,
                                              C.c_void_p(want.ctypes.data), C.byref(pts), H))
    cols = [np.full(N, np.nan) for _ in range(nb * p)]
    carr = (C.c_void_p * (nb * p))(*[c.ctypes.data for c in cols])
    pq._lib.check(pq._lib.lib.pq_phi_adaptive_cols(ctx.handle, d, sh, fac, nb, barr, p, 1e-10, carr, C.byref(pts2), H))
    assert np.array_equal(np.stack(cols).reshape(nb, p, N), want) and pts.value == pts2.value
    exps = np.concatenate([pq.expm(np.ascontiguousarray(f), scale=[0.25], ctx=ctx)[0].reshape(-1) for f in w.factors])
    y = np.ascontiguousarray(want[0])
    y2 = [np.ascontiguousarray(want[0, j]) for j in range(p)]
    pq._lib.check(pq._lib.lib.pq_squaring_step(ctx.handle, d, sh, exps.ctypes.data_as(pq._lib.dp), p,
                                               C.c_void_p(y.ctypes.data), H))
    yarr = (C.c_void_p * p)(*[c.ctypes.data for c in y2])
    pq._lib.check(pq._lib.lib.pq_squaring_step_cols(ctx.handle, d, sh, exps.ctypes.data_as(pq._lib.dp), p, yarr, H))
    assert np.array_equal(np.stack(y2), y)
    ctx.close()
