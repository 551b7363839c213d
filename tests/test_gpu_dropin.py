"""Runs the C++ drop-in example (reference-style user code linked to the
sm_100a library) on the GPU."""
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_cpp_dropin_example_runs(cuda):
    from paper_2504_13821_b200 import build as b

    exe = b.build_dropin_example()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dropin_example: ok" in r.stdout


@pytest.mark.parametrize("storage", ["buffer", "pageable"])
def test_dropin_bench_host_storages(cuda, storage):
    """Reference-caller-shaped e2e: rec_trsm<double> on MatrixBuffers (the
    drop-in allocates them page-locked) and on plain std::vector storage
    behind MatrixViews (pageable, through the pinned bounce staging) -- the
    residual gate must pass (exit 0) and the timing line must parse."""
    import json

    from paper_2504_13821_b200 import build as b

    exe = b.build_dropin_bench()
    r = subprocess.run([str(exe), "2048", "3000", "2", "1", storage], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["storage"] == storage
    assert d["finite"] and d["eta"] <= 32 and len(d["step_ms"]) == 2


def test_matrixbuffer_storage_is_page_locked(cuda):
    """rectri_cu_host_alloc (the drop-in MatrixBuffer's allocator) returns
    page-locked memory on a GPU box, plain memory with
    RECTRI_CU_PINNED_BUFFERS=0; rectri_cu_host_free releases both."""
    import ctypes

    from paper_2504_13821_b200 import _lib

    lib = _lib.load()
    lib.rectri_cu_host_alloc.restype = ctypes.c_void_p
    lib.rectri_cu_host_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(ctypes.c_int32)]
    lib.rectri_cu_host_free.argtypes = [ctypes.c_void_p]
    pinned = ctypes.c_int32(-1)
    p = lib.rectri_cu_host_alloc(1 << 20, ctypes.byref(pinned))
    assert p and pinned.value == 1
    ctypes.memset(p, 0, 1 << 20)
    lib.rectri_cu_host_free(p)
