"""Error conventions of the C ABI: invalid arguments return
MDC_EINVAL (-22) before any device work, with a message in the calling
thread's mdc_last_error(); the Python wrapper turns a negative status into
MdcError.  Argument validation precedes every CUDA call, so this runs on CPU."""
import ctypes
import threading

import pytest

from paper_1408_0677_b200 import _lib

EINVAL = -22
FAKE = 0x1000  # a 16-byte-aligned non-null "device pointer" (never dereferenced: validation fails first)


def _err(lib):
    return lib.mdc_last_error().decode()


def _mls_args(**kw):
    a = _lib.MdcMlsArgs()
    a.variant, a.dtype = _lib.MDC_AFFINE, _lib.MDC_F32
    a.width, a.height, a.row0, a.row1 = 8, 8, 0, 8
    a.n, a.d, a.ldq = 4, 4, 4
    a.pc = a.q = a.qm = a.out = FAKE
    for k, v in kw.items():
        setattr(a, k, v)
    return a


@pytest.mark.parametrize("kw,msg", [
    (dict(variant=7), "variant"),
    (dict(dtype=3), "dtype"),
    (dict(width=0), "width/height"),
    (dict(row0=5, row1=4), "row band"),
    (dict(row1=9), "row band"),
    (dict(n=0), "control"),
    (dict(d=0), "channel"),
    (dict(variant=_lib.MDC_RIGID, d=3, ldq=4), "rigid"),
    (dict(variant=_lib.MDC_MEAN), "axis"),
    (dict(out=None), "null device pointer"),
    (dict(bands=FAKE), "spacing"),
    (dict(ldq=3), "ldq"),
    (dict(ldq=5), "ldq"),
    (dict(q=FAKE + 4), "aligned"),
    (dict(rgba=FAKE), "palette"),
    (dict(rgba=FAKE, spacing=FAKE), "palette"),
    (dict(rgba=FAKE, spacing=FAKE, palette=FAKE, palette_n=0), "palette"),
])
def test_mls_field_rejects_bad_arguments(kw, msg):
    lib = _lib.load()
    assert lib.mdc_mls_field(ctypes.byref(_mls_args(**kw)), None) == EINVAL
    assert msg in _err(lib)


def test_other_entry_points_reject_bad_arguments():
    lib = _lib.load()
    assert lib.mdc_mls_field(None, None) == EINVAL and "null args" in _err(lib)
    assert lib.mdc_pca(1, 4, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, None) == EINVAL and "n >= 2" in _err(lib)
    la = _lib.MdcLayoutArgs()
    la.n, la.leaf = 0, 32
    h = ctypes.c_void_p()
    assert lib.mdc_layout_plan_create(ctypes.byref(la), ctypes.byref(h), None) == EINVAL and "n out of range" in _err(lib)
    assert lib.mdc_layout_set_gather(None, FAKE) == EINVAL and "null" in _err(lib)
    assert lib.mdc_layout_scatter(None, FAKE, 1, None) == EINVAL and "null" in _err(lib)
    assert lib.mdc_rigid_field_norm(1, FAKE, FAKE, 2, FAKE, FAKE, FAKE, FAKE, 1.0, FAKE, None, None) == EINVAL
    assert "norm_out" in _err(lib)
    la.n, la.leaf = 10, 0
    assert lib.mdc_layout_plan_create(ctypes.byref(la), ctypes.byref(h), None) == EINVAL and "leaf" in _err(lib)
    la.leaf = 32
    assert lib.mdc_layout_plan_create(ctypes.byref(la), ctypes.byref(h), None) == EINVAL and "topology" in _err(lib)
    ra = _lib.MdcRenderArgs()
    ra.values = ra.spacing = ra.out = FAKE
    ra.mode = 9
    assert lib.mdc_render(ctypes.byref(ra), None) == EINVAL and "render mode" in _err(lib)
    assert lib.mdc_mls_prepare(0, 1, FAKE, FAKE, _lib.MDC_AFFINE, _lib.MDC_F32, None, 4, FAKE, FAKE, FAKE, FAKE,
                               FAKE, 1 << 20, None) == EINVAL and "bad sizes" in _err(lib)


def test_wrapper_raises_mdc_error_with_the_message():
    lib = _lib.load()
    rc = lib.mdc_mls_field(ctypes.byref(_mls_args(n=0)), None)
    with pytest.raises(_lib.MdcError, match=r"mdc_mls_field failed \(-22\): .*control"):
        _lib.check(rc, "mdc_mls_field")


def test_last_error_is_thread_local():
    lib = _lib.load()
    seen, go = {}, threading.Barrier(2)

    def worker(name, kw):
        go.wait()
        for _ in range(200):
            assert lib.mdc_mls_field(ctypes.byref(_mls_args(**kw)), None) == EINVAL
            seen.setdefault(name, set()).add(_err(lib))

    t1 = threading.Thread(target=worker, args=("dtype", dict(dtype=3)))
    t2 = threading.Thread(target=worker, args=("width", dict(width=0)))
    t1.start(), t2.start()
    t1.join(), t2.join()
    assert len(seen["dtype"]) == 1 and "dtype" in next(iter(seen["dtype"]))
    assert len(seen["width"]) == 1 and "width/height" in next(iter(seen["width"]))
