"""Generates tests/golden/*.json from the UNMODIFIED reference (oracle/_ref, built from /root/reference/proj).

Run in the build container (the reference sources are not on the GPU box):

    python tools/make_golden.py

The fixtures pin the CPU oracle (oracle/gempe_oracle.c), the product's host numerics and, on the GPU, the
CUDA path.  Every value below is an output of a public symbol of the reference library; nothing is typed in.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2011_03479_b200.graphgen import Stream  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def ring(n):
    s = np.arange(n, dtype=np.uint32)
    return n, s, ((s + 1) % n).astype(np.uint32)


def er_graph(n, m, seed):
    rng = Stream(seed, 77)
    chosen = {}
    while len(chosen) < m:
        a, b = (int(v) for v in rng.below(2, n))
        if a == b:
            continue
        chosen.setdefault((min(a, b), max(a, b)), None)
    e = np.array(list(chosen), np.uint32)
    return n, np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])


def dump(name, obj):
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(obj, f, separators=(",", ":"))
    print(name, os.path.getsize(os.path.join(OUT, name)), "bytes")


def main():
    ref = O.Ref()
    L = ref.lib
    rng = Stream(20260101, 5)

    # ---- integer layer ---------------------------------------------------------------------------
    ints = {"splitmix64": [], "mix_seed": [], "expand_seed32": [], "lane_uniform_index": [], "pair_hash": []}
    for v in [0, 1, 2, 0xdeadbeef] + [int(x) for x in rng.u64(12)]:
        ints["splitmix64"].append([str(v), str(L.ref_splitmix64(v))])
    for _ in range(16):
        s, c = (int(x) for x in rng.u64(2))
        c >>= int(rng.below(1, 60)[0])
        ints["mix_seed"].append([str(s), str(c), str(L.ref_mix_seed(s, c))])
    ints["mix_seed"].append(["1", str(0xA11BE11), str(L.ref_mix_seed(1, 0xA11BE11))])
    for args in [(1, 0, 0, 0), (1, 0, 0, 1), (1, 0, 1, 0), (42, 3, 7, 1)]:
        ints["expand_seed32"].append([*map(str, args), L.ref_expand_seed32(*args)])
    for _ in range(24):
        s = int(rng.u64(1)[0])
        a, b, c = (int(x) for x in rng.below(3, 1 << 28))
        ints["expand_seed32"].append([str(s), str(a), str(b), str(c), L.ref_expand_seed32(s, a, b, c)])
    ns = [1, 2, 3, 97, 1000, 3000, 100000, 1 << 20, (1 << 23) - 1, 1 << 23, (1 << 23) + 1, (1 << 23) + 12345,
          1 << 24, 3000000000]
    words = [0, 0xff800000, 0x007fffff, 0xffffffff, 12345678, 0xdeadbeef] + [int(x) & 0xffffffff for x in rng.u64(26)]
    for n in ns:
        for w in words:
            ints["lane_uniform_index"].append([w, n, L.ref_lane_uniform_index(w, n)])
    cases = [(0, 0, 77, 1 << 20), (0, 1, 2, 1 << 20), (70000, 70001, 1 << 17, 1 << 20), (5, 9, 3000, 1 << 21),
             (1048575, 1048574, 1 << 20, 1 << 30)]
    for _ in range(200):
        i, j, n = (int(x) & 0xffffffff for x in rng.u64(3))
        cases.append((i, j, n, 1 << (1 + int(rng.below(1, 31)[0]))))
    for i, j, n, size in cases:
        ints["pair_hash"].append([i, j, n, size, L.ref_pair_hash(i, j, n, size)])
    dump("integer_layer.json", ints)

    # ---- FastMath tables, parabola, sigma optimiser -------------------------------------------------
    num = {"tables": {}, "ratio": [], "parabola": [], "sigma": []}
    for which, name in [(0, "erf"), (1, "exp_neg"), (2, "ratio")]:
        flat, odd = ref.fastmath_table(which)
        num["tables"][name] = {"flat": [repr(float(v)) for v in flat], "odd_mirror": int(odd)}
    for x in np.concatenate([np.linspace(-8, 12, 81), [-6.0, -1.0, 8.0, 8.000001, 25.0, -0.9999, 5.5]]):
        num["ratio"].append([repr(float(x)), repr(L.ref_gauss_erfc_ratio(float(x), 1)),
                             repr(L.ref_gauss_erfc_ratio(float(x), 0))])
    for sigma in [1e-3, 0.05, 0.3, 1.0, 1.5, 3.7, 16.0]:
        for delta in [0.0, 1e-6, 0.1, 0.5, 1.0, 1.5, 2.0, 3.0, 5.0, 9.0, 12.0, 40.0]:
            for is_edge in (1, 0):
                row = [repr(delta), repr(sigma), is_edge]
                for fast in (1, 0):
                    d, w = ref.parabola(delta, 1.5, sigma, is_edge, fast)
                    row += [repr(d), repr(w)]
                num["parabola"].append(row)
    for case in range(6):
        he = np.zeros(512, np.uint64)
        hn = np.zeros(512, np.uint64)
        centre_e, centre_n = 20 + 15 * case, 60 + 40 * case
        for b in rng.below(400 + 300 * case, 60):
            he[min(511, centre_e + int(b) - 30 if centre_e + int(b) - 30 > 0 else 0)] += 1
        for b in rng.below(800 + 500 * case, 200):
            hn[min(511, centre_n + int(b) - 60 if centre_n + int(b) - 60 > 0 else 0)] += 1
        nw = 3.0 + 50.0 * case
        s, steps = ref.optimize_sigma(he, hn, nw, 1.5)
        num["sigma"].append({
            "edge": [int(v) for v in he], "nonedge": [int(v) for v in hn], "nonedge_weight": nw,
            "sigma": repr(s), "steps": steps,
            "objective": repr(L.ref_histogram_objective(he, hn, nw, 1.5, s)),
            "dsigma_at_1": repr(L.ref_histogram_objective_dsigma(he, hn, nw, 1.5, 1.0))})
    dump("numerics.json", num)

    # ---- relabel / init ---------------------------------------------------------------------------------
    prep = {"relabel": [], "init": []}
    for n, seed in [(1, 5), (2, 5), (8, L.ref_mix_seed(1, 0xA11BE11)), (50, 123456789), (257, 2**63 + 11)]:
        prep["relabel"].append({"n": n, "seed": str(seed), "forward": [int(v) for v in ref.random_relabel(n, seed)]})
    for n, dim, seed in [(5, 2, 1), (3, 7, 99), (4, 128, 2**40 + 3)]:
        x = ref.init_embedding(n, dim, seed)
        prep["init"].append({"n": n, "dim": dim, "seed": str(seed), "bits": [int(v) for v in x.view(np.uint32).ravel()]})
    dump("prep.json", prep)

    # ---- engine traces ----------------------------------------------------------------------------------
    traces = []
    cases = [("ring8_d2", ring(8), 2, 1, True, 3), ("er120_d2_exact", er_graph(120, 400, 31), 2, 14, False, 3),
             ("er60_d5", er_graph(60, 150, 7), 5, 3, True, 2), ("er40_d16", er_graph(40, 90, 9), 16, 21, True, 2)]
    for name, (n, src, dst), dim, seed, fast, iters in cases:
        eng = O.RefEngine(ref, n, src, dst, dim, seed, lane_width=16, workers=2, fast_math=fast)
        ws, wd = eng.work_graph()
        hs = O.RefHash(ref, n, ws, wd)
        case = {"name": name, "n": n, "dim": dim, "seed": seed, "fast_math": int(fast), "src": [int(v) for v in src],
                "dst": [int(v) for v in dst], "work_src": [int(v) for v in ws], "work_dst": [int(v) for v in wd],
                "hash_size": eng.hash_size, "x0_bits": [int(v) for v in eng.work_coords().view(np.uint32).ravel()],
                "rounds": []}
        i = rng.below(400, n).astype(np.uint32)
        j = rng.below(400, n).astype(np.uint32)
        case["probe"] = {"i": [int(v) for v in i], "j": [int(v) for v in j], "out": [int(v) for v in eng.probe(i, j)]}
        for it in range(iters):
            sigma_in = eng.sigma
            m = len(ws)
            anchors = np.empty(2 * m, np.uint32)
            states = np.empty(2 * m, np.uint32)
            for e in range(m):
                for draw in (0, 1):
                    anchors[2 * e + draw] = ws[e] if draw == 0 else wd[e]
                    states[2 * e + draw] = L.ref_expand_seed32(seed, it, e, draw)
            rc, partners, _, draws = hs.sample(anchors, states)
            assert rc == 0
            out = eng.iterate()
            case["rounds"].append({
                "sigma_in": repr(sigma_in), "partners": [int(v) for v in partners], "draws": int(draws),
                "y": [repr(float(v)) for v in out["y"].ravel()], "z": [repr(float(v)) for v in out["z"]],
                "x_bits": [int(v) for v in eng.work_coords().view(np.uint32).ravel()],
                "sigma_out": repr(out["sigma"]), "pe_estimate": repr(out["pe_estimate"])})
        traces.append(case)
    dump("engine_traces.json", traces)

    # ---- full embed() runs ---------------------------------------------------------------------------------
    runs = []
    for name, (n, src, dst), dim, seed, max_iters in [("er97", er_graph(97, 400, 13), 2, 4, 40),
                                                       ("ring12", ring(12), 2, 6, 25)]:
        eng = O.RefEngine(ref, n, src, dst, dim, seed, lane_width=16, workers=3, max_iters=max_iters)
        res = eng.run()
        runs.append({"name": name, "n": n, "dim": dim, "seed": seed, "max_iters": max_iters,
                     "src": [int(v) for v in src], "dst": [int(v) for v in dst],
                     "iterations": res["iterations"], "converged": int(res["converged"]),
                     "final_sigma": repr(res["final_sigma"]), "pe_trace": [repr(float(v)) for v in res["pe_trace"]],
                     "hist_edge_total": int(res["hist_edge"].sum()), "hist_nonedge_total": int(res["hist_nonedge"].sum()),
                     "relabel_forward": [int(v) for v in res["relabel_forward"]],
                     "embedding": [repr(float(v)) for v in res["embedding"].ravel()]})
    dump("embed_runs.json", runs)

    # ---- text formats: edge-list canonicalisation, snapshot bytes, TSV export ------------------------------
    import base64
    fm = {"edge_lists": [], "tsv": [], "snapshots": []}
    texts = ["0 1\n1 2\n", "0 0\n0 1\n1 0\n", "5 9\n9 7\n", "# header\n% more\n\n   \n0 1\n", "0 1\n2 x\n", "0 1 2\n",
             "7\n", "-1 2\n", "3 3\n", "# only comments\n", "5 9\n9 7\n7 5\n1 5\n", "10\t20\r\n20 30\r\n30   10", "",
             "18446744073709551615 1\n18446744073709551616 2\n", "1 2\n\n\n2 1\n3 1 \n  4\t3\n", "1 2\n 3 4 x\n",
             "9 8\n8 9\n9 9\n7 8", "0 1\x00\n", "4 5\n#6 7\n %8 9\n6 7 \v\f\n"]
    soup = Stream(1, 99)
    for _ in range(40):
        ln = int(soup.below(1, 120)[0])
        texts.append(bytes(int(v) for v in soup.below(ln, 256)).decode("latin1"))
    for _ in range(40):  # digit-rich soup that often parses
        ln = int(soup.below(1, 80)[0])
        alphabet = "0123456789  \n\n\t#%x"
        texts.append("".join(alphabet[int(v)] for v in soup.below(ln, len(alphabet))))
    for t in texts:
        raw = t.encode("latin1")
        r = ref.load_edge_list(raw)
        entry = {"text_b64": base64.b64encode(raw).decode(), "rc": r["rc"]}
        if r["rc"] == 0:
            entry.update(n=r["n"], src=[int(v) for v in r["src"]], dst=[int(v) for v in r["dst"]],
                         labels=[str(int(v)) for v in r["labels"]])
        else:
            entry.update(line=r.get("line", 0), error=r["error"])
        fm["edge_lists"].append(entry)
    emb = ref.init_embedding(3, 2, 5)
    fm["tsv"].append({"n": 3, "dim": 2, "bits": [int(v) for v in emb.view(np.uint32).ravel()], "labels": ["42", "7", "100"],
                      "perm": None, "text": ref.write_embedding_tsv(emb, [42, 7, 100]).decode()})
    emb = ref.init_embedding(4, 1, 9)
    fm["tsv"].append({"n": 4, "dim": 1, "bits": [int(v) for v in emb.view(np.uint32).ravel()], "labels": None,
                      "perm": [2, 3, 0, 1], "text": ref.write_embedding_tsv(emb, None, [2, 3, 0, 1]).decode()})
    emb = (ref.init_embedding(6, 5, 77) - 0.5) * np.float32(1e4)
    emb[0, 0], emb[1, 1], emb[2, 2] = 0.0, 1e-7, -123456789.0
    fm["tsv"].append({"n": 6, "dim": 5, "bits": [int(v) for v in emb.view(np.uint32).ravel()],
                      "labels": ["9", "3", "1000000000000", "0", "5", "4"], "perm": [5, 4, 3, 2, 1, 0],
                      "text": ref.write_embedding_tsv(emb, [9, 3, 10**12, 0, 5, 4], [5, 4, 3, 2, 1, 0]).decode()})
    n_, s_, d_ = er_graph(20, 40, 3)
    fm["snapshots"].append({"n": n_, "src": [int(v) for v in s_], "dst": [int(v) for v in d_],
                            "bytes_b64": base64.b64encode(ref.save_graph_snapshot(n_, s_, d_)).decode()})
    dump("formats.json", fm)


if __name__ == "__main__":
    main()
