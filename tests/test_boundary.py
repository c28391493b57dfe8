"""C-ABI boundary checks that need no GPU: the in-tree sm_100a library
loads, exports every entry point include/rcpg.h declares, the ctypes layer
binds exactly those, config structs have the C layout, and the product path
never touches the oracle (the checker)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rcpg.h")
PKG = os.path.join(ROOT, "paper_1703_09074_b200")


def header_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rcpg_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_reference_surface():
    syms = header_symbols()
    for must in ["rcpg_decompose", "rcpg_compress", "rcpg_relative_error", "rcpg_tensor_upload", "rcpg_create"]:
        assert must in syms


def test_library_exports_every_header_symbol(rcp):
    from paper_1703_09074_b200 import _lib
    assert os.path.exists(_lib.LIB_PATH), "build the extension first (__graft_entry__.build())"
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (rcpg_[a-z_0-9]+)\b", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing


def test_ctypes_binds_exactly_the_header(rcp):
    from paper_1703_09074_b200 import _lib
    assert sorted(_lib.SIGNATURES) == header_symbols()
    L = _lib.lib()
    assert L.rcpg_version().decode().startswith("rcpg")


def test_library_is_sm100a_native():
    from paper_1703_09074_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_struct_layout(rcp, tmp_path):
    """ctypes mirrors must have the C compiler's layout of include/rcpg.h."""
    from paper_1703_09074_b200 import _lib
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "rcpg.h"\nint main(void){'
                   'printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(rcpg_compress_config), '
                   'offsetof(rcpg_compress_config, modes), offsetof(rcpg_compress_config, seed), '
                   'sizeof(rcpg_decompose_config), offsetof(rcpg_decompose_config, compress), '
                   'offsetof(rcpg_decompose_config, tol), sizeof(rcpg_result)); return 0;}')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [C.sizeof(_lib.CompressConfigC), _lib.CompressConfigC.modes.offset, _lib.CompressConfigC.seed.offset,
            C.sizeof(_lib.DecomposeConfigC), _lib.DecomposeConfigC.compress.offset, _lib.DecomposeConfigC.tol.offset,
            C.sizeof(_lib.ResultC)]
    assert got == want


def test_product_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "pyoracle" not in text and "rcp_oracle" not in text and "liboracle" not in text, f


def test_no_gpu_fails_loudly(rcp):
    """Without a device the context cannot be created and the API raises (no
    silent CPU fallback)."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(rcp.CudaError):
        rcp.Context(0)


def test_derive_seed_and_stream_ids_match_oracle(rcp, oracle):
    for seed in [0, 1, 42, 2**63 + 5]:
        for salt in [0, 7, (1 << 32) | 3]:
            assert rcp.derive_seed(seed, salt) == oracle.derive_seed(seed, salt)
    assert rcp.stream_id(rcp.COMPRESS, 2) == oracle.stream_id(1, 2)


@pytest.mark.parametrize("kind,shape,rank", [(1, [12, 10, 9], 3), (2, [12, 10, 9], 4), (3, [12, 10, 9], 4),
                                             (4, [12, 10, 9, 7], 3), (5, [12, 10, 9], 4)])
def test_synthetic_models_match_oracle_generators(rcp, oracle, kind, shape, rank):
    from paper_1703_09074_b200 import synthetic
    w, f = synthetic.model(kind, shape, rank, 3)
    if kind == 1:
        _, (wo, fo) = oracle.random_lowrank(shape, rank, 3)
        # the reference normalizes the truth model; the tensor is the same
        xo = oracle.reconstruct(wo, fo)
        x = oracle.reconstruct(w, f)
        assert np.max(np.abs(x - xo)) <= 1e-12 * np.max(np.abs(xo))
        return
    _, (wo, fo) = oracle.synth(kind, shape, rank, 3, 0.0)
    assert np.max(np.abs(w - wo)) <= 1e-14 * np.max(np.abs(wo))
    for a, b in zip(f, fo):
        assert np.max(np.abs(a - b)) <= 1e-12


def test_synthetic_normals_are_the_reference_stream(rcp, oracle):
    from paper_1703_09074_b200 import synthetic
    sid = oracle.stream_id(4)
    got = synthetic.normals(17, sid, 1001)
    want = oracle.stream_draws(17, sid, "normal", 1001)
    assert np.max(np.abs(got - want)) <= 4 * np.spacing(np.abs(want)).max()
