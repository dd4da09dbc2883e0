"""Host-buffer path of pq_phi_0p with PINNED output buffers: phi_0 is copied out on the side stream
while the squaring runs (capi.cpp run_phiquadmv).  The results must equal the device-resident path
bitwise and be complete when the call returns (no later synchronisation by the caller)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [16, 64])
def test_pinned_host_outputs_equal_device_outputs(pq, n):
    import torch
    from paper_2211_00696_b200.workloads import config
    w = config(2, n=n)
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
    pq._lib.check(pq._lib.lib.pq_phi_0p(ctx.handle, d, sh, fac, 1, C.c_void_p(b_pin.data_ptr()), C.byref(rc),
                                        C.c_void_p(o0_pin.data_ptr()), C.c_void_p(o_pin.data_ptr()), C.byref(info),
                                        pq._lib.PQ_HOST))
    # read immediately: the call must have completed every copy it issued
    assert np.array_equal(o0_pin.numpy(), o0_dev.cpu().numpy())
    assert np.array_equal(o_pin.numpy(), o_dev.cpu().numpy())
    ctx.close()
