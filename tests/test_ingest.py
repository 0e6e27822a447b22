"""Edge-list ingest against the reference's own parser.

The product reader (csrc/host/ingest.cpp: mmap + chunked parallel scan +
bitmap id compaction) must accept exactly what proj/src/graph.cpp:54-99
accepts, build the same graph, and report the same first bad line with the
same message.  The reference runs here from oracle/_ref (lrref_graph_parse).
"""
import os
import tempfile

import numpy as np
import pytest

from oracle_py import Ref


@pytest.fixture(scope="module")
def ref():
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    return Ref()


def _ours(lr, data, dense):
    try:
        g = lr.Graph.parse_edge_list(data, dense_ids=dense)
    except OSError as e:
        return ("err", str(e))
    return ("ok", g.n, g.csr()[:2])


def _theirs(ref, data, dense):
    try:
        g = ref.parse(data, dense)
    except ValueError as e:
        return ("err", str(e))
    return ("ok", g.n, g.csr()[:2])


def _same(a, b):
    if a[0] != b[0]:
        return False
    if a[0] == "err":
        return a[1] == b[1]
    return a[1] == b[1] and all(np.array_equal(x, y) for x, y in zip(a[2], b[2]))


# the reference's own parse cases (proj/tests/test_graph.cpp:54-102), restated
CASES = [
    b"# header\n0\t1\r\n2\t3\n\n1\t2\n",
    b"5\t9\n9\t100\n",
    b"0 1\n", b"0\t1\na\tb\n", b"0\t\n", b"0\t1\n0\t1\ttrailing\n", b"-1\t0\n",
    b"# only a comment\n", b"", b"\n\n", b"0\t1", b"0\t1\r", b"0\t1\r\r\n", b"\t1\n", b"1\t\t2\n",
    b"+1\t2\n", b"-0\t3\n", b"007\t8\n", b"2147483647\t0\n",
    b"9223372036854775807\t1\n", b"9223372036854775808\t1\n", b"-9223372036854775808\t1\n",
    b"99999999999999999999999\t1\n", b"1\t2 \n", b" 1\t2\n", b"#\t\n3\t3\n", b"1\t2\n#x\n\r\n2\t1\n",
    b"3\t4\n3\t4\n4\t4\n", b"-\t1\n", b"1\t-\n", b"1\t-2\n",
]


# ids up to kMaxVertexId are legal; with dense ids they would make 2^31-vertex
# graphs, so they are checked with compaction only
SPARSE_ONLY = [b"2147483646\t0\n", b"1\t2147483646\n2147483646\t5\n"]


@pytest.mark.parametrize("dense", [True, False])
def test_reference_parse_cases(lr, ref, dense):
    for data in CASES + ([] if dense else SPARSE_ONLY):
        a, b = _ours(lr, data, dense), _theirs(ref, data, dense)
        assert _same(a, b), (data, a, b)


def test_fuzzed_lines(lr, ref):
    rng = np.random.default_rng(7)
    tokens = ["0", "1", "7", "12", "305", "007", "-", "-1", "-0", "\t", "\t", "\t", "\n", "\n", "\n", "\r", "#",
              " ", "a", "2147483647", "99999999999999999999"]
    for t in range(600):
        k = int(rng.integers(0, 24))
        data = "".join(rng.choice(tokens, size=k)).encode()
        for dense in (True, False):
            a, b = _ours(lr, data, dense), _theirs(ref, data, dense)
            assert _same(a, b), (data, a, b)


def _big_text(rng, lines, n):
    s = rng.integers(0, n, lines)
    d = rng.integers(0, n, lines)
    body = [f"{x}\t{y}" for x, y in zip(s, d)]
    for i in rng.choice(lines, lines // 50, replace=False):  # comments, blanks, CRLF sprinkled in
        body[i] = ["# c", "", body[i] + "\r"][i % 3]
    return body


def test_multi_chunk_buffers(lr, ref):
    """Inputs of tens of MB run on every host thread: same graph, and an error
    planted deep in the file is reported at its global line number."""
    rng = np.random.default_rng(11)
    body = _big_text(rng, 3_000_000, 5_000_000)
    data = ("\n".join(body) + "\n").encode()
    assert len(data) > 8 << 22
    for dense in (True, False):
        assert _same(_ours(lr, data, dense), _theirs(ref, data, dense))
    for at in (2_999_999, 1_700_000, 400_000):
        bad = list(body)
        bad[at] = "12\tx"
        bad[at + 1 if at + 1 < len(bad) else at - 1] = "oops"
        data = ("\n".join(bad) + "\n").encode()
        a, b = _ours(lr, data, True), _theirs(ref, data, True)
        assert a[0] == "err" and _same(a, b), (a, b)


def test_load_edge_list_mmap(lr, ref):
    rng = np.random.default_rng(3)
    data = ("\n".join(_big_text(rng, 200_000, 300_000)) + "\n").encode()
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "g.tsv")
        with open(p, "wb") as f:
            f.write(data)
        g = lr.Graph.load_edge_list(p, dense_ids=False)
        r = ref.parse(data, False)
        assert g.n == r.n
        assert all(np.array_equal(x, y) for x, y in zip(g.csr()[:2], r.csr()[:2]))
        open(os.path.join(d, "empty.tsv"), "wb").close()
        with pytest.raises(OSError, match="empty input"):
            lr.Graph.load_edge_list(os.path.join(d, "empty.tsv"))
        with pytest.raises(OSError, match="cannot open"):
            lr.Graph.load_edge_list(os.path.join(d, "missing.tsv"))
