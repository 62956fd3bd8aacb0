"""Graph ingest and embedding export (host side of the path) against the committed outputs of
the reference's load_edge_list / save_graph_snapshot / write_embedding_tsv.  CPU only."""
import base64
import os

import numpy as np
import pytest

from conftest import load_golden


def test_edge_list_canonicalisation_matches_reference():
    from paper_2011_03479_b200 import engine as E
    cases = load_golden("formats.json")["edge_lists"]
    assert sum(c["rc"] == 0 for c in cases) >= 10 and sum(c["rc"] == 5 for c in cases) >= 10
    for c in cases:
        text = base64.b64decode(c["text_b64"])
        if c["rc"] == 0:
            g, labels = E.load_edge_list(text)
            assert g.n == c["n"] and g.src.tolist() == c["src"] and g.dst.tolist() == c["dst"]
            assert [str(int(v)) for v in labels] == c["labels"]
        elif c["rc"] == 5:  # parse_error carries the 1-based line
            with pytest.raises(E.ParseError) as err:
                E.load_edge_list(text)
            assert err.value.line == c["line"]
        else:  # data_error: nothing survived canonicalisation
            with pytest.raises(E.DataError) as err:
                E.load_edge_list(text)
            assert not isinstance(err.value, E.ParseError)


def test_reference_loader_cases_by_hand():
    """tests/test_graph.cpp:34-91 restated."""
    from paper_2011_03479_b200 import engine as E
    g, labels = E.load_edge_list("5 9\n9 7\n")
    assert (g.n, g.src.tolist(), g.dst.tolist(), labels.tolist()) == (3, [0, 1], [1, 2], [5, 9, 7])
    g, _ = E.load_edge_list("0 0\n0 1\n1 0\n")
    assert (g.n, g.edge_count()) == (2, 1)
    with pytest.raises(E.ParseError) as err:
        E.load_edge_list("0 1\n2 x\n")
    assert err.value.line == 2
    for bad in ("0 1 2\n", "7\n", "-1 2\n"):
        with pytest.raises(E.ParseError):
            E.load_edge_list(bad)
    for empty in ("3 3\n", "# only comments\n"):
        with pytest.raises(E.DataError):
            E.load_edge_list(empty)
    # load / emit idempotence
    g, _ = E.load_edge_list("5 9\n9 7\n7 5\n1 5\n")
    emitted = "".join(f"{a}\t{b}\n" for a, b in zip(g.src.tolist(), g.dst.tolist()))
    g2, _ = E.load_edge_list(emitted)
    assert g2.n == g.n and np.array_equal(g2.src, g.src) and np.array_equal(g2.dst, g.dst)


def test_snapshot_bytes_and_round_trip(tmp_path):
    from paper_2011_03479_b200 import engine as E, graphgen
    for snap in load_golden("formats.json")["snapshots"]:
        want = base64.b64decode(snap["bytes_b64"])
        g = E.Graph(snap["n"], snap["src"], snap["dst"])
        path = str(tmp_path / "g.gemp")
        E.save_graph_snapshot(path, g)
        assert open(path, "rb").read() == want
        back = E.load_graph_snapshot(want)
        assert back.n == g.n and np.array_equal(back.src, g.src) and np.array_equal(back.dst, g.dst)
        g3, labels = E.load_graph_file(path)  # magic sniffing (embed_main.cpp:150-153)
        assert g3.n == g.n and labels is None and np.array_equal(g3.dst, g.dst)
        n2, s2, d2 = graphgen.load_snapshot(path)  # the numpy reader agrees
        assert n2 == g.n and np.array_equal(s2, g.src)
    txt = str(tmp_path / "e.txt")
    open(txt, "w").write("0 1\n")
    assert E.load_graph_file(txt)[0].edge_count() == 1
    for bad in (b"GEMX" + bytes(20), b"GEMP" + bytes(4), b"GEMP" + (3).to_bytes(4, "little") + (0).to_bytes(8, "little"),
                b"GEMP" + (3).to_bytes(4, "little") + (9).to_bytes(8, "little") + bytes(72),
                b"GEMP" + (3).to_bytes(4, "little") + (1).to_bytes(8, "little") + (1).to_bytes(4, "little") * 2):
        with pytest.raises(E.DataError):
            E.load_graph_snapshot(bad)


def test_embedding_tsv_matches_reference_text(tmp_path):
    from paper_2011_03479_b200 import engine as E
    for c in load_golden("formats.json")["tsv"]:
        x = np.array(c["bits"], np.uint32).view(np.float32).reshape(c["n"], c["dim"])
        labels = None if c["labels"] is None else [int(v) for v in c["labels"]]
        path = str(tmp_path / "emb.tsv")
        E.write_embedding_tsv(path, x, labels, c["perm"])
        assert open(path).read() == c["text"]
    with pytest.raises(E.DataError):
        E.write_embedding_tsv(str(tmp_path / "x.tsv"), np.zeros((3, 2), np.float32), [1, 2])
