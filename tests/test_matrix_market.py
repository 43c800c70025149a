"""CPU: MatrixMarket ingest (generators.read_matrix_market, C++ host code)
against the reference's reader (matrix_market.cpp:48-132) on the same files,
bit for bit, plus its error contract and a write/read round trip."""
import numpy as np
import pytest

from paper_1801_03065_b200 import generators as G

GENERAL = """%%MatrixMarket matrix coordinate real general
% a comment

3 4 6
1 1 1.5
3 4 -2.25e-3
% interleaved comment
2 2 7
1 1 0.25
1 3 1e300

3 1 -0
"""

SYMMETRIC = """%%MatrixMarket matrix coordinate real symmetric
4 4 5
1 1 2.0
2 1 -1.0
3 2 -1.0
4 3 -1.0
4 4 2.0
"""

PATTERN = """%%MatrixMarket matrix coordinate pattern general
2 3 3
1 3
2 1
1 3
"""

INTEGER = """%%MatrixMarket matrix coordinate integer symmetric
3 3 2
2 1 5
3 3 -4
"""

BAD = {
    "header": "%%MatrixMarket tensor coordinate real general\n1 1 1\n1 1 1\n",
    "array": "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "field": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "range": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n",
    "short": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n",
    "value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 x\n",
}


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def _same(a, b):
    assert (a.num_rows, a.num_cols) == (b.num_rows, b.num_cols)
    assert np.array_equal(a.row_offsets, b.row_offsets)
    assert np.array_equal(a.col_indices, b.col_indices)
    assert np.array_equal(np.asarray(a.values).view(np.int64), np.asarray(b.values).view(np.int64))


def test_general_with_comments_and_duplicates(tmp_path):
    m = G.read_matrix_market(_write(tmp_path, "g.mtx", GENERAL))
    assert (m.num_rows, m.num_cols) == (3, 4)
    assert m.row_offsets.tolist() == [0, 2, 3, 5]
    assert m.col_indices.tolist() == [0, 2, 1, 0, 3]
    assert m.values.tolist() == [1.75, 1e300, 7.0, -0.0, -2.25e-3]


def test_symmetric_pattern_integer(tmp_path):
    s = G.read_matrix_market(_write(tmp_path, "s.mtx", SYMMETRIC))
    assert s.nnz() == 8 and s.row_offsets.tolist() == [0, 2, 4, 6, 8]
    p = G.read_matrix_market(_write(tmp_path, "p.mtx", PATTERN))
    assert p.col_indices.tolist() == [2, 0] and p.values.tolist() == [2.0, 1.0]
    i = G.read_matrix_market(_write(tmp_path, "i.mtx", INTEGER))
    assert i.values.tolist() == [5.0, 5.0, -4.0]


@pytest.mark.parametrize("kind", sorted(BAD))
def test_errors(tmp_path, kind):
    with pytest.raises(ValueError):
        G.read_matrix_market(_write(tmp_path, kind + ".mtx", BAD[kind]))
    with pytest.raises(ValueError):
        G.read_matrix_market(str(tmp_path / "missing.mtx"))


def test_round_trip(tmp_path):
    a = G.laplace2d(9)
    path = str(tmp_path / "rt.mtx")
    G.write_matrix_market(a, path)
    _same(G.read_matrix_market(path), a)


def test_matches_reference_reader(tmp_path, reference):
    for name, text in (("g", GENERAL), ("s", SYMMETRIC), ("p", PATTERN), ("i", INTEGER)):
        path = _write(tmp_path, name + ".mtx", text)
        _same(G.read_matrix_market(path), reference.read_mm(path))
    a = G.rmat(8, 4, 3)
    path = str(tmp_path / "rmat.mtx")
    G.write_matrix_market(a, path)
    _same(G.read_matrix_market(path), reference.read_mm(path))
    for kind in sorted(BAD):
        with pytest.raises(ValueError):
            reference.read_mm(_write(tmp_path, kind + "_ref.mtx", BAD[kind]))


def test_multi_slice_file_matches_reference(tmp_path, reference):
    """A file large enough to be tokenised in several slices (one per host
    thread) reads bit-identically to the reference reader, symmetric too."""
    a = G.rmat(14, 16, 5)
    path = str(tmp_path / "big.mtx")
    G.write_matrix_market(a, path)
    _same(G.read_matrix_market(path), reference.read_mm(path))
    # symmetric: lower triangle of a, mirrored on read
    lines = ["%%MatrixMarket matrix coordinate real symmetric"]
    ents = []
    for i in range(a.num_rows):
        for q in range(int(a.row_offsets[i]), int(a.row_offsets[i + 1])):
            j = int(a.col_indices[q])
            if j <= i:
                ents.append(f"{i + 1} {j + 1} {float(a.values[q]):.17g}")
    lines.append(f"{a.num_rows} {a.num_cols} {len(ents)}")
    sym = str(tmp_path / "sym.mtx")
    with open(sym, "w") as f:
        f.write("\n".join(lines + ents) + "\n")
    _same(G.read_matrix_market(sym), reference.read_mm(sym))


def test_entries_after_the_declared_count_are_ignored(tmp_path, reference):
    text = "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n2 2 2\n9 9 garbage\n"
    path = _write(tmp_path, "extra.mtx", text)
    m = G.read_matrix_market(path)
    assert m.nnz() == 2 and m.values.tolist() == [1.0, 2.0]
    _same(m, reference.read_mm(path))


def test_error_line_numbers(tmp_path):
    text = "%%MatrixMarket matrix coordinate real general\n% c\n3 3 3\n1 1 1\n\n2 2 x\n3 3 3\n"
    with pytest.raises(ValueError, match="line 6"):
        G.read_matrix_market(_write(tmp_path, "ln.mtx", text))
