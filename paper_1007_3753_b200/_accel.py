"""The native kernel seam of the reference (ell1._accel, _accel/__init__.py:1-27,
_fastkernels.pyx:14-78), served by libell1b200.so on the GPU.

Same functions, argument contracts and side effects:
  soft_threshold(u, a)  -> new float64 array     (u: 1-d C-contiguous float64)
  project_box_linf(z)   -> new float64 array
  chol_update(R, v)     -> 0; R (m x m C-contiguous) updated IN PLACE, v consumed
  chol_downdate(R, v)   -> 0 or failing pivot + 1; R, v modified in place
There is no fallback backend: COMPILED is True, and a missing library or
device raises DeviceError at the first call.
"""

import numpy as np

from paper_1007_3753_b200 import _lib, device

COMPILED = True


def _vec(u, name):
    if not isinstance(u, np.ndarray) or u.dtype != np.float64 or u.ndim != 1 or not u.flags.c_contiguous:
        raise ValueError("%s must be a 1-d C-contiguous float64 array" % name)
    return u


def soft_threshold(u, a):
    _vec(u, "u")
    L = _lib.lib()
    torch = device._torch()
    dev = device.current_device()
    n = u.shape[0]
    if n == 0:
        return np.empty(0)
    ud = torch.from_numpy(u).to(dev)
    od = torch.empty_like(ud)
    _lib.check(L.ell1_soft_threshold(device.ptr(ud), float(a), device.ptr(od), n, device.stream_ptr(dev)),
               "ell1_soft_threshold")
    return od.cpu().numpy()


def project_box_linf(z):
    _vec(z, "z")
    L = _lib.lib()
    torch = device._torch()
    dev = device.current_device()
    n = z.shape[0]
    if n == 0:
        return np.empty(0)
    zd = torch.from_numpy(z).to(dev)
    od = torch.empty_like(zd)
    _lib.check(L.ell1_project_box_linf(device.ptr(zd), device.ptr(od), n, device.stream_ptr(dev)),
               "ell1_project_box_linf")
    return od.cpu().numpy()


def _rank1(fn, R, v):
    if not isinstance(R, np.ndarray) or R.dtype != np.float64 or R.ndim != 2 or not R.flags.c_contiguous:
        raise ValueError("R must be a 2-d C-contiguous float64 array")
    _vec(v, "v")
    m = R.shape[0]
    if R.shape[1] != m or v.shape[0] < m:
        raise ValueError("R must be square and v at least as long as R")
    torch = device._torch()
    dev = device.current_device()
    if m == 0:
        return 0
    Rd = torch.from_numpy(R).to(dev)
    vd = torch.from_numpy(v).to(dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(fn(device.ptr(Rd), device.ptr(vd), m, device.ptr(st), device.stream_ptr(dev)), "chol rank-1")
    R[...] = Rd.cpu().numpy()
    v[:m] = vd.cpu().numpy()[:m]
    return int(st.item())


def chol_update(R, v):
    return _rank1(_lib.lib().ell1_chol_update, R, v)


def chol_downdate(R, v):
    return _rank1(_lib.lib().ell1_chol_downdate, R, v)
