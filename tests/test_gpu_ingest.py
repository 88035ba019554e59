"""GPU matrix ingestion (SURVEY §8(a) A2 from_coo, §8(f) rank 4 Matrix Market): bit-identical to
the reference's from_coo (csr.hpp:72-110) and read_matrix_market (matrix_market.hpp:48-113),
checked against the compiled reference and the oracle restatement."""
import numpy as np
import pytest

import paper_2309_02228_b200 as mpkg
from conftest import assert_bitwise

pytestmark = pytest.mark.gpu


def _same(dev, ref):
    n_rows, n_cols, rp, ci, v = ref
    H = dev.download()
    assert (H.n_rows, H.n_cols) == (n_rows, n_cols)
    np.testing.assert_array_equal(H.row_ptr, rp)
    np.testing.assert_array_equal(H.col_idx, ci)
    assert_bitwise(H.values, v)


def test_from_coo_duplicates_signed_zeros_empty_rows(ctx, oracle, ref):
    rng = np.random.default_rng(3)
    for trial in range(25):
        nr, nc = int(rng.integers(1, 300)), int(rng.integers(1, 300))
        m = int(rng.integers(0, 3000))
        r = rng.integers(0, nr, m).astype(np.uint32)
        c = rng.integers(0, nc, m).astype(np.uint32)
        # duplicates with cancellation, lone -0.0 entries (0.0 + -0.0 = +0.0 in the reference)
        v = rng.choice([-0.0, 1.0, -1.0, 1e-300, 3.5, -3.5, 1e300], m) * rng.uniform(0.5, 2, m)
        v[rng.random(m) < 0.05] = -0.0
        got = ctx.csr_from_coo(nr, nc, r, c, v)
        _same(got, ref.from_coo(nr, nc, r, c, v))
        orp, oci, ov = oracle.from_coo(nr, nc, r, c, v)
        np.testing.assert_array_equal(got.download().row_ptr, orp)


def test_from_coo_large_and_errors(ctx, ref):
    rng = np.random.default_rng(5)
    n, m = 200_000, 3_000_000
    r = rng.integers(0, n, m).astype(np.uint32)
    c = rng.integers(0, n, m).astype(np.uint32)
    v = rng.uniform(-1, 1, m)
    _same(ctx.csr_from_coo(n, n, r, c, v), ref.from_coo(n, n, r, c, v))
    with pytest.raises(ValueError, match=r"out of range at \(5, 7\)"):
        ctx.csr_from_coo(4, 10, [0, 5, 9], [1, 7, 0], [1.0, 2.0, 3.0])


def _write(path, text):
    path.write_bytes(text.encode())
    return path


def test_matrix_market_variants(ctx, ref, tmp_path):
    rng = np.random.default_rng(11)
    cases = []
    for sym in ("general", "symmetric", "skew-symmetric"):
        for field in ("real", "integer", "pattern"):
            n = 40
            ents = set()
            while len(ents) < 150:
                i, j = int(rng.integers(1, n + 1)), int(rng.integers(1, n + 1))
                if sym != "general" and j > i:
                    i, j = j, i
                if sym == "skew-symmetric" and i == j:
                    continue
                ents.add((i, j))
            eol = "\r\n" if sym == "symmetric" else "\n"
            # a blank line is only skipped when truly empty: with CRLF it is "\r" (the reference
            # then fails on it, see test_matrix_market_errors)
            lines = [f"%%MatrixMarket Matrix Coordinate {field.upper()} {sym}", "% a comment"]
            lines += ([] if eol == "\r\n" else [""]) + [f"{n} {n} {len(ents) + 2}"]
            for k, (i, j) in enumerate(sorted(ents)):
                if field == "pattern":
                    lines.append(f"{i} {j}")
                elif field == "integer":
                    lines.append(f"{i} {j} {int(rng.integers(-9, 10))}")
                else:
                    lines.append(f"{i}  {j}\t{rng.uniform(-1, 1):.17g}")
                if k == 10:
                    lines.append("% comment between entries")
            i0, j0 = sorted(ents)[0]
            for _ in range(2):  # duplicates of the first entry (summed in line order)
                lines.append(f"{i0} {j0}" + ("" if field == "pattern" else " 0.125"))
            cases.append(_write(tmp_path / f"m_{sym}_{field}.mtx", eol.join(lines) + eol))
    cases.append(_write(tmp_path / "rect.mtx", "%%MatrixMarket matrix coordinate real general\n"
                                                "3 5 4\n1 5 1e-310\n3 1 -2.5E3\n2 2 .5\n1 5 7\n"))
    for path in cases:
        _same(ctx.read_matrix_market(path), ref.read_matrix_market(path))


@pytest.mark.parametrize("text,msg", [
    ("", "empty file"),
    ("%%MatrixMarket matrix array real general\n1 1\n1\n", "unsupported banner"),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n", "unsupported field"),
    ("%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n", "unsupported symmetry"),
    ("%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1\n", "missing banner"),
    ("%%MatrixMarket matrix coordinate real general\n2 x 1\n", "malformed size line"),
    ("%%MatrixMarket matrix coordinate real general\n0 2 1\n", "empty dimensions"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "fewer entries"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", "out of range"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n", "missing value"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 inf\n", "missing value"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1e400\n", "missing value"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\nx 1 1.0\n", "malformed entry"),
    ("%%MatrixMarket matrix coordinate real general\r\n\r\n2 2 1\r\n1 1 1.0\r\n", "malformed size line"),
])
def test_matrix_market_errors(ctx, ref, tmp_path, text, msg):
    path = _write(tmp_path / "bad.mtx", text)
    with pytest.raises(RuntimeError, match=msg):
        ref.read_matrix_market(path)
    with pytest.raises(mpkg.MpkgError, match=msg):
        ctx.read_matrix_market(path)
    with pytest.raises(mpkg.MpkgError, match="cannot open"):
        ctx.read_matrix_market(tmp_path / "missing.mtx")
