"""The matrix file format (matrix_io.hpp:14-77) and the command line front end
(tools/qgemm_main.cpp) on the GPU path. Spec: the reference's
tests/test_io.cpp and tests/test_cli.cpp, restated; the parser and writer are
also pinned byte for byte against the reference's own read_matrix /
write_matrix (oracle/_ref) where it is built. CLI cases that multiply are
marked gpu; plan inspection, usage and parse errors need no device."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

import oracle as O
import paper_0803_1975_b200 as qg

needs_ref = pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built here")


def splitmix(seed):
    state = seed
    while True:
        state = (state + 0x9E3779B97F4A7C15) & (2**64 - 1)
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        yield z ^ (z >> 31)


def ref_write(m, p):
    m = np.ascontiguousarray(m, np.uint32)
    rows, cols = m.shape
    need = O.REF.qgref_write_matrix(m.ctypes.data_as(ctypes.c_void_p), rows, cols, p, None, 0)
    buf = ctypes.create_string_buffer(need + 1)
    O.REF.qgref_write_matrix(m.ctypes.data_as(ctypes.c_void_p), rows, cols, p, buf, need)
    return buf.raw[:need].decode()


def ref_parse(text):
    raw = text.encode()
    p, rows, cols = ctypes.c_uint32(), ctypes.c_size_t(), ctypes.c_size_t()
    data = np.zeros(4096, np.uint32)
    msg = ctypes.create_string_buffer(512)
    st = O.REF.qgref_parse_matrix(raw, len(raw), ctypes.byref(p), ctypes.byref(rows), ctypes.byref(cols),
                                  data.ctypes.data_as(ctypes.c_void_p), data.size, msg, 512)
    if st:
        return st, msg.value.decode()
    return st, (p.value, data[: rows.value * cols.value].reshape(rows.value, cols.value))


def ours_parse(text):
    try:
        return 0, qg.parse_matrix(text)
    except qg.ParseError as e:
        return 8, str(e)


# ------------------------------------------------------------------ test_io.cpp
def test_matrix_files_round_trip(tmp_path):  # test_io.cpp:11-23
    rng = splitmix(17)
    for trial in range(25):
        rows, cols = next(rng) % 12, next(rng) % 12
        m = O.random_residue_matrix(rows, cols, 11, trial + 500)
        path = str(tmp_path / f"m{trial}.mtx")
        qg.write_matrix_file(path, m, 11)
        p, got = qg.read_matrix_file(path)
        assert p == 11 and got.shape == (rows, cols) and np.array_equal(got, m)
        if O.REF is not None:
            assert open(path).read() == ref_write(m, 11)


@pytest.mark.parametrize("text", ["X 3 1 1\n0\n", "M 1 1 1\n0\n", "M 3 2 2\n0 1 2\n", "M 3 1 2\n0 3\n",
                                  "M 3 1 2\n0 1 2\n", "M 3 1 -2\n"])
def test_parser_rejects_malformed_input(text):  # test_io.cpp:25-37
    with pytest.raises(qg.ParseError):
        qg.parse_matrix(text)


def test_parser_accepts_an_empty_body():
    p, m = qg.parse_matrix("M 3 0 4\n")
    assert p == 3 and m.shape == (0, 4)


@needs_ref
def test_parser_matches_the_reference_on_edge_and_fuzzed_inputs():
    cases = ["M 3 2 2\n0 1\n2 0\n", "M 3 2 2 0 1 2 0", "M\t5\n1\n3\n4 0 1\n", "M 3 1 2\n+1 2\n", "M 3 1 2\n01 2\n",
             "M 3 1 2\n1 2abc\n", "M 3 1 2\n1 2 junk\n", "M 3 1 2\n1 2 -0\n", "M 3 1 1\n-0\n", "M 3 1 1\n4294967296\n",
             "M 4294967296 1 1\n0\n", "M 3 1 1 1\n", "M 3 1\n", "", "M", "m 3 1 1\n0\n", "M 3 1 1\n0x1\n",
             "M 7 2 3\n6 5 4\n3 2 1\n\n\n", "M 2 0 0\n", "M 2 0 0 1\n", "M 3 1 2\n1\t2\r\n", "M 3 1 1\n99999999999999999999\n"]
    rng = np.random.default_rng(5)
    alphabet = list("M 0123456789-+\nx\t")
    for _ in range(300):
        cases.append("".join(rng.choice(alphabet, size=int(rng.integers(1, 24)))))
    for text in cases:
        st_ref, ref = ref_parse(text)
        st, ours = ours_parse(text)
        assert st == st_ref, (text, ref, ours)
        if st == 0:
            assert ours[0] == ref[0] and np.array_equal(ours[1], ref[1]), text
        else:
            assert ours == ref, text


def test_unreadable_file_is_a_parse_error():
    with pytest.raises(qg.ParseError, match="cannot open"):
        qg.read_matrix_file("/nonexistent/dir/m.mtx")


# ------------------------------------------------------------------ test_cli.cpp
def run_cli(*args):
    r = subprocess.run([qg.CLI_PATH, *args], capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout + r.stderr


def test_cli_plan():  # test_cli.cpp:58-78
    rc, out = run_cli("plan", "--p", "3", "--k", "200", "--bits", "53")
    assert rc == 0 and "Q        2^10" in out and "e        5" in out
    rc, out = run_cli("plan", "--p", "3", "--k", "200", "--bits", "53", "--full")
    assert rc == 0 and "dq+1     2" in out and "dtheta+1 2" in out
    assert run_cli("plan", "--p", "100003", "--k", "10")[0] == 3
    assert run_cli("plan", "--p", "4", "--k", "10")[0] == 2
    assert run_cli("plan", "--k", "10")[0] == 2


@needs_ref
def test_cli_plan_prints_the_reference_plans():
    for p, k, beta in [(3, 200, 53), (7, 4096, 53), (5, 8192, 63), (2, 1, 53), (13, 1000, 40)]:
        rc, out = run_cli("plan", "--p", str(p), "--k", str(k), "--bits", str(beta))
        pl = O.Plan()
        st = O.REF.qgref_plan_compression(p, k, beta, 0, ctypes.byref(pl))
        assert (rc == 0) == (st == 0)
        if st == 0:
            want = f"p        {p}\nk        {k}\nbeta     {pl.beta}\nt        {pl.t}\nQ        2^{pl.t}\n" \
                   f"d        {pl.d}\ne        {pl.e}\nkmax     {pl.kmax}\n"
            assert out == want


def test_cli_help_and_usage():  # test_cli.cpp:164-169
    assert run_cli("--help")[0] == 0
    assert run_cli()[0] == 2
    assert run_cli("frobnicate")[0] == 2
    assert run_cli("plan", "--p", "3", "--k")[0] == 2
    assert run_cli("plan", "--p", "three", "--k", "5")[0] == 2
    assert run_cli("verify", "--p", "4", "--max-dim", "8", "--seeds", "5")[0] == 2  # test_cli.cpp:125-126


def test_cli_gemm_input_errors(tmp_path):  # test_cli.cpp:109-118 (no product is run)
    a = O.random_residue_matrix(9, 14, 3, 1)
    b = O.random_residue_matrix(14, 7, 3, 2)
    ap, bp, out = str(tmp_path / "a.mtx"), str(tmp_path / "b.mtx"), str(tmp_path / "o.mtx")
    qg.write_matrix_file(ap, a, 3)
    qg.write_matrix_file(bp, b, 3)
    rc, msg = run_cli("gemm", "--algo", "common", "--a", bp, "--b", ap, "--out", out)
    assert rc == 2 and "14x7" in msg and "9x14" in msg
    assert run_cli("gemm", "--algo", "common", "--a", "/nonexistent.mtx", "--b", bp, "--out", out)[0] == 2
    qg.write_matrix_file(str(tmp_path / "b5.mtx"), b % 2, 5)
    assert run_cli("gemm", "--algo", "common", "--a", ap, "--b", str(tmp_path / "b5.mtx"), "--out", out)[0] == 2
    assert run_cli("gemm", "--algo", "common", "--a", ap, "--b", bp, "--out", out, "--p", "5")[0] == 2
    assert run_cli("gemm", "--a", ap, "--b", bp, "--out", out)[0] == 2


@pytest.mark.gpu
def test_cli_gemm(tmp_path):  # test_cli.cpp:80-107
    a = O.random_residue_matrix(9, 14, 3, 1)
    b = O.random_residue_matrix(14, 7, 3, 2)
    ap, bp = str(tmp_path / "a.mtx"), str(tmp_path / "b.mtx")
    qg.write_matrix_file(ap, a, 3)
    qg.write_matrix_file(bp, b, 3)
    naive_out = str(tmp_path / "naive.mtx")
    assert run_cli("gemm", "--algo", "naive", "--a", ap, "--b", bp, "--out", naive_out)[0] == 0
    p, want = qg.read_matrix_file(naive_out)
    assert p == 3 and np.array_equal(want, O.naive_gemm(3, a, b))
    for algo in ("common", "right", "left", "full", "blocked"):
        out = str(tmp_path / f"{algo}.mtx")
        rc, msg = run_cli("gemm", "--algo", algo, "--a", ap, "--b", bp, "--out", out)
        assert rc == 0, msg
        assert np.array_equal(qg.read_matrix_file(out)[1], want), algo
    eye = np.eye(14, dtype=np.uint32)
    qg.write_matrix_file(str(tmp_path / "eye.mtx"), eye, 3)
    eye_out = str(tmp_path / "eye_out.mtx")
    assert run_cli("gemm", "--algo", "naive", "--a", str(tmp_path / "eye.mtx"), "--b", bp, "--out", eye_out)[0] == 0
    assert np.array_equal(qg.read_matrix_file(eye_out)[1], b)
    # a common dimension past the plan's reach: infeasible (3), blocked works
    big_a = O.random_residue_matrix(5, 70000, 3, 3)
    big_b = O.random_residue_matrix(70000, 4, 3, 4)
    qg.write_matrix_file(str(tmp_path / "ba.mtx"), big_a, 3)
    qg.write_matrix_file(str(tmp_path / "bb.mtx"), big_b, 3)
    rc, msg = run_cli("gemm", "--algo", "full", "--a", str(tmp_path / "ba.mtx"), "--b", str(tmp_path / "bb.mtx"),
                      "--out", str(tmp_path / "bo.mtx"))
    assert rc == 3 and "blocked" in msg
    rc, _ = run_cli("gemm", "--algo", "blocked", "--a", str(tmp_path / "ba.mtx"), "--b", str(tmp_path / "bb.mtx"),
                    "--out", str(tmp_path / "bo.mtx"))
    assert rc == 0 and np.array_equal(qg.read_matrix_file(str(tmp_path / "bo.mtx"))[1], O.naive_gemm(3, big_a, big_b))


@pytest.mark.gpu
def test_cli_verify():  # test_cli.cpp:120-127
    rc, out = run_cli("verify", "--p", "3", "--max-dim", "8", "--seeds", "5")
    assert rc == 0 and "common" in out and "blocked" in out and "ok" in out and "FAIL" not in out
    assert run_cli("verify", "--p", "2", "--max-dim", "4", "--seeds", "3")[0] == 0
    rc, out = run_cli("verify", "--p", "7", "--max-dim", "40", "--seeds", "30")
    assert rc == 0 and out.count("ok") == 10, out  # 5 algorithms x {double, int64}


@pytest.mark.gpu
def test_cli_bench():  # test_cli.cpp:129-154
    rc, out = run_cli("bench", "--p", "3", "--m", "16", "--k", "16", "--n", "16", "--algo", "common", "--reps", "3",
                      "--seed", "9")
    assert rc == 0, out
    lines = out.strip().split("\n")
    assert lines[0] == "algorithm,p,m,k,n,t,e,seconds_multiply,seconds_convert,checksum"
    assert len(lines) == 4
    want = O.residue_checksum(O.naive_gemm(3, O.random_residue_matrix(16, 16, 3, 9), O.random_residue_matrix(16, 16, 3, 10)))
    pl = O.plan_compression(3, 16)
    for row in lines[1:]:
        f = row.split(",")
        assert f[:7] == ["common", "3", "16", "16", "16", str(pl.t), str(pl.e)]
        assert int(f[9]) == want
    for algo in ("naive", "right", "left", "full", "blocked"):
        rc, out = run_cli("bench", "--p", "3", "--m", "16", "--k", "16", "--n", "16", "--algo", algo, "--seed", "9")
        assert rc == 0, out
        assert int(out.strip().split("\n")[1].split(",")[9]) == want, algo
    assert run_cli("bench", "--p", "100003", "--m", "8", "--k", "8", "--n", "8", "--algo", "common", "--reps", "1",
                   "--seed", "1")[0] == 3


@pytest.mark.gpu
def test_cli_int64_backend(tmp_path):
    """--bits 54..63 runs the Int64Word backend (qgemm_main.cpp:253-266); verify
    checks both backends (verify.hpp:128-137)."""
    rc, out = run_cli("verify", "--p", "3", "--max-dim", "12", "--seeds", "8")
    assert rc == 0, out
    lines = [l for l in out.strip().split("\n") if l]
    assert len(lines) == 10 and sum("\tint64\t" in l for l in lines) == 5, out
    assert all("\tok (" in l for l in lines)
    a = O.random_residue_matrix(9, 300, 3, 1)
    b = O.random_residue_matrix(300, 7, 3, 2)
    ap, bp = str(tmp_path / "a.mtx"), str(tmp_path / "b.mtx")
    qg.write_matrix_file(ap, a, 3)
    qg.write_matrix_file(bp, b, 3)
    want = O.naive_gemm(3, a, b)
    for algo in ("common", "right", "left", "full", "blocked"):
        out = str(tmp_path / f"{algo}64.mtx")
        rc, msg = run_cli("gemm", "--algo", algo, "--a", ap, "--b", bp, "--out", out, "--bits", "63")
        assert rc == 0, (algo, msg)
        assert np.array_equal(qg.read_matrix_file(out)[1], want), algo
    rc, out = run_cli("bench", "--p", "3", "--m", "16", "--k", "200", "--n", "16", "--algo", "common", "--bits", "63",
                      "--seed", "9")
    assert rc == 0, out
    pl = O.plan_compression(3, 200, 63)
    f = out.strip().split("\n")[1].split(",")
    assert f[5:7] == [str(pl.t), str(pl.e)]
    assert int(f[9]) == O.residue_checksum(O.naive_gemm(3, O.random_residue_matrix(16, 200, 3, 9),
                                                        O.random_residue_matrix(200, 16, 3, 10)))
