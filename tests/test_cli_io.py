"""CLI and file formats either side of the path:
the reference's DTEN / KTEN layouts (proj/include/rcp/io.hpp:92-189, written
here byte by byte with struct, independent of the C++ code under test), their
error messages, the canonical-form rule for models (io.hpp:135-137 ->
kruskal.hpp:117-176, checked against the oracle's normalize), the trace CSV,
and the `rcp` CLI (proj/tools/main.cpp): options, summary line, exit codes."""
import os
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1703_09074_b200")
CLI = os.path.join(LIBDIR, "rcp")


def dten(shape, values, dtype=0, version=1, magic=b"DTEN"):
    v = np.ascontiguousarray(values, dtype=np.float64 if dtype == 0 else np.float32)
    return magic + bytes([version, dtype, len(shape)]) + b"".join(struct.pack("<Q", e) for e in shape) + v.tobytes()


def kten(weights, factors, version=1):
    out = b"KTEN" + bytes([version]) + struct.pack("<QQ", len(weights), len(factors))
    out += b"".join(struct.pack("<Q", f.shape[0]) for f in factors)
    out += np.asarray(weights, dtype=np.float64).tobytes()
    for f in factors:
        out += np.ascontiguousarray(f, dtype=np.float64).tobytes()  # row-major (io.hpp:62-69)
    return out


@pytest.fixture(scope="module")
def io_main(tmp_path_factory, rcp):
    exe = tmp_path_factory.mktemp("io") / "io_main"
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "io_main.cpp"), "-L", LIBDIR, "-lrcpg",
                    f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    return str(exe)


def run(*args):
    return subprocess.run([str(a) for a in args], capture_output=True, text=True, timeout=600)


def test_tensor_roundtrip_is_byte_identical(io_main, tmp_path):
    rng = np.random.default_rng(0)
    for shape, dt in [((3, 4, 5), 0), ((2, 3, 4, 2), 0), ((7,), 0), ((3, 4, 5), 1)]:
        src, dst = tmp_path / "a.dten", tmp_path / "b.dten"
        blob = dten(shape, rng.standard_normal(shape), dtype=dt)
        src.write_bytes(blob)
        r = run(io_main, "tensor", src, dst)
        assert r.returncode == 0, r.stderr
        assert dst.read_bytes() == blob


@pytest.mark.parametrize("blob,msg", [
    (dten((2, 2), np.ones(4), magic=b"XTEN"), "read_tensor: bad magic, not a tensor file"),
    (dten((2, 2), np.ones(4), version=2), "read_tensor: unsupported version 2"),
    (dten((2, 2), np.ones(4), dtype=0)[:4] + bytes([1, 7, 2]) + dten((2, 2), np.ones(4))[7:], "read_tensor: unsupported dtype 7"),
    (b"DTEN" + bytes([1, 0, 0]), "read_tensor: order must be at least 1"),
    (dten((2, 0), np.ones(0)), "read_tensor: invalid extent"),
    (dten((2, 2), np.ones(4))[:-3], "truncated file while reading payload"),
    (dten((2, 2), np.ones(4)) + b"\x00", "read_tensor: trailing bytes after payload"),
    (dten((2, 2), np.array([1.0, np.nan, 0.0, 1.0])), "read_tensor: non-finite values"),
])
def test_tensor_reader_errors_match_reference(io_main, tmp_path, blob, msg):
    src = tmp_path / "bad.dten"
    src.write_bytes(blob)
    r = run(io_main, "tensor", src, tmp_path / "out.dten")
    assert r.returncode == 1 and r.stderr.strip() == f"error: {msg}", r.stderr


def test_model_canonical_form_and_roundtrip(io_main, oracle, tmp_path):
    rng = np.random.default_rng(3)
    shape, R = (5, 4, 3), 4
    w = np.array([2.0, -3.0, 0.5, 3.0])
    fs = [rng.standard_normal((e, R)) for e in shape]
    fs[1][:, 2] = 0.0  # zero column -> e1, weight 0
    src, dst, dst2 = tmp_path / "m.kten", tmp_path / "n.kten", tmp_path / "o.kten"
    src.write_bytes(kten(w, fs))
    r = run(io_main, "model", src, dst)
    assert r.returncode == 0, r.stderr
    wn, fn = oracle.normalize(w, [np.asfortranarray(f) for f in fs])
    want = kten(wn, fn)
    got = dst.read_bytes()
    hdr = 5 + 8 * (2 + 3)  # magic, version, rank, order, extents
    assert len(got) == len(want) and got[:hdr] == want[:hdr]
    g = np.frombuffer(got[hdr:], dtype=np.float64)
    h = np.frombuffer(want[hdr:], dtype=np.float64)
    assert np.max(np.abs(g - h)) <= 1e-15
    r = run(io_main, "model", dst, dst2)  # canonical input is written back unchanged
    assert r.returncode == 0 and dst2.read_bytes() == got


@pytest.mark.parametrize("blob,msg", [
    (b"KTEX" + bytes(40), "read_kruskal: bad magic, not a model file"),
    (kten([1.0], [np.ones((2, 1))], version=3), "read_kruskal: unsupported version 3"),
    (b"KTEN" + bytes([1]) + struct.pack("<QQ", 0, 2), "read_kruskal: implausible rank or order"),
    (kten([1.0], [np.ones((2, 1))])[:-8], "truncated file while reading factor"),
    (kten([np.inf], [np.ones((2, 1))]), "read_kruskal: non-finite weights"),
])
def test_model_reader_errors_match_reference(io_main, tmp_path, blob, msg):
    src = tmp_path / "bad.kten"
    src.write_bytes(blob)
    r = run(io_main, "model", src, tmp_path / "out.kten")
    assert r.returncode == 1 and r.stderr.strip() == f"error: {msg}", r.stderr


def test_trace_csv_format(io_main, tmp_path):
    out = tmp_path / "t.csv"
    assert run(io_main, "trace", out).returncode == 0
    assert out.read_text() == "iteration,fit,seconds\n1,0.5,0.25\n2,0.75,0.5\n"


def test_cli_usage_and_errors(rcp, tmp_path):
    assert os.path.exists(CLI), "built by __graft_entry__.build()"
    assert run(CLI, "--help").returncode == 0
    assert run(CLI).returncode == 1
    assert run(CLI, "frobnicate").returncode == 1
    r = run(CLI, "decompose", "--in", tmp_path / "x.dten", "--out", tmp_path / "m.kten")
    assert r.returncode == 1 and "--rank is required" in r.stderr
    r = run(CLI, "decompose", "--in", tmp_path / "x.dten", "--rank", "3", "--out", tmp_path / "m.kten", "--bogus", "1")
    assert r.returncode == 1 and "not expected" in r.stderr
    r = run(CLI, "decompose", "--in", tmp_path / "x.dten", "--rank", "3", "--out", tmp_path / "m.kten",
            "--deterministic", "--power-iters", "1")
    assert r.returncode == 1
    r = run(CLI, "decompose", "--in", tmp_path / "missing.dten", "--rank", "3", "--out", tmp_path / "m.kten")
    assert r.returncode == 1 and r.stderr.strip() == f"error: cannot open for reading: {tmp_path / 'missing.dten'}"


@pytest.mark.gpu
def test_cli_synth_decompose_reconstruct_match_the_api(rcp, oracle, tmp_path):
    x, mt, tr, rec = tmp_path / "x.dten", tmp_path / "m.kten", tmp_path / "fit.csv", tmp_path / "truth.kten"
    r = run(CLI, "synth", "--shape", "40,30,20", "--rank", "5", "--snr", "10", "--seed", "7", "--out", x, "--truth", rec)
    assert r.returncode == 0, r.stderr
    blob = x.read_bytes()
    assert blob[:7] == b"DTEN" + bytes([1, 0, 3])
    data = np.frombuffer(blob[7 + 24:], dtype=np.float64).reshape(40, 30, 20)
    want, _ = oracle.random_lowrank([40, 30, 20], 5, 7, snr=10.0, noise_seed=7)
    assert np.max(np.abs(data - want)) <= 1e-12 * np.max(np.abs(want))  # device libm vs glibc: ulps
    r = run(CLI, "decompose", "--in", x, "--rank", "5", "--seed", "7", "--tol", "1e-8", "--max-iter", "100",
            "--out", mt, "--trace", tr)
    assert r.returncode == 0, r.stdout + r.stderr
    fields = dict(kv.split("=") for kv in r.stdout.split())
    assert fields["method"] == "als" and fields["randomized"] == "true" and fields["rank"] == "5"
    cs = rcp.derive_seed(7, rcp.stream_id(rcp.COMPRESS))
    cfg = rcp.DecomposeConfig(rank=5, tol=1e-8, max_iter=100, seed=7,
                              compress=rcp.CompressConfig(target_rank=5, oversampling=10, power_iterations=2, seed=cs))
    model, trace = rcp.decompose(data, cfg)
    assert int(fields["iters"]) == trace.iterations
    assert abs(float(fields["error"]) - trace.final_relative_error) <= 1e-11
    m = mt.read_bytes()
    w = np.frombuffer(m[45:45 + 8 * 5], dtype=np.float64)  # after magic, version, rank, order, 3 extents
    assert np.array_equal(w, model.weights)
    lines = tr.read_text().splitlines()
    assert lines[0] == "iteration,fit,seconds" and len(lines) == trace.iterations + 1
    out = tmp_path / "xhat.dten"
    r = run(CLI, "reconstruct", "--in", mt, "--out", out)
    assert r.returncode == 0, r.stderr
    xhat = np.frombuffer(out.read_bytes()[31:], dtype=np.float64).reshape(40, 30, 20)
    ref = oracle.reconstruct(model.weights, [np.asfortranarray(f) for f in model.factors])
    assert np.max(np.abs(xhat - ref)) <= 1e-12 * np.max(np.abs(ref))
    # not converged within max_iter -> exit code 2
    r = run(CLI, "decompose", "--in", x, "--rank", "5", "--max-iter", "1", "--out", mt)
    assert r.returncode == 2, r.stdout + r.stderr
