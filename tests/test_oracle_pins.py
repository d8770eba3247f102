"""Pins for the CPU oracle (marked not-gpu).  The oracle is trusted only because
these tests tie it to things other than itself (task ③): the SPEC worked
examples (tests/golden), brute force over all injective maps, networkx VF2
monomorphisms, and closed forms (SURVEY.md §8(c) "What pins each part").

A plausible mistake in the oracle — a dropped edge check, a missing
injectivity test, a wrong label index, a transposed row — fails at least one
of: brute force (every definition clause), closed forms on K_n (injectivity),
star/P4 labeled forms (labels), C4 codegree form (non-tree edge checks),
row-level equality (column order)."""
import itertools
import json
import os

import numpy as np
import pytest

import gsm_inputs as gi
import oracle
from oracle import closed_forms as cf

HERE = os.path.dirname(os.path.abspath(__file__))


def _graph(d):
    g = gi.from_edge_list(d["num_nodes"], d["edges"])
    if "labels" in d:
        g = g.with_labels(np.asarray(d["labels"], np.uint32))
    return g


def _query(d):
    return gi.Query(d["num_nodes"], [tuple(e) for e in d["edges"]], d.get("labels"))


# ------------------------------------------------------------------ golden (SPEC)
def test_spec_golden_examples():
    ex = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))["examples"]
    assert len(ex) >= 8
    for e in ex:
        g, q = _graph(e["data"]), _query(e["query"])
        cnt, rows = oracle.match(g, q)
        assert cnt == e["all"] == len(rows), e["cite"]
        aut = oracle.automorphisms(q)
        uniq = oracle.unique(rows, aut)
        assert len(uniq) == e["unique"], e["cite"]
        if "unique_node_sets" in e:
            assert sorted(sorted(r) for r in uniq.tolist()) == e["unique_node_sets"]
        if "aut_size" in e:
            assert len(aut) == e["aut_size"]


# ------------------------------------------------------------------ brute force
def _tiny_instances():
    out = []
    for seed in range(1, 13):
        n = 6 + seed % 3
        g = gi.random_gnp(n, 1, 2, seed)
        for k, extra in [(2, 0), (3, 1), (4, 1), (4, 2), (5, 2)]:
            for nl in (0, 2):
                q = gi.random_connected_query(k, extra, seed * 31 + k + extra, nl)
                gg = g.with_labels(gi.uniform_labels(n, 2, seed)) if nl else g
                out.append((gg, q))
    return out


def test_oracle_equals_brute_force():
    inst = _tiny_instances()
    assert len(inst) >= 100
    nonzero = 0
    for g, q in inst:
        cnt, rows = oracle.match(g, q)
        bf = oracle.brute_force(g, q)
        assert cnt == len(bf)
        np.testing.assert_array_equal(rows, bf)
        nonzero += cnt > 0
    assert nonzero > 40  # the instances are not all trivially empty


def test_brute_force_is_the_definition():
    # pin the brute force itself on K_4 (every injective map is an embedding)
    assert len(oracle.brute_force(gi.complete(4), gi.query("K3"))) == 24
    assert len(oracle.brute_force(gi.cycle(4), gi.query("K3"))) == 0
    assert len(oracle.brute_force(gi.path(3), gi.query("K2"))) == 4


# ------------------------------------------------------------------ networkx VF2
def _nx(g):
    import networkx as nx
    G = nx.Graph()
    G.add_nodes_from(range(g.num_nodes))
    src = np.repeat(np.arange(g.num_nodes), np.diff(g.offsets))
    G.add_edges_from(zip(src.tolist(), g.cols.tolist()))
    if g.labels is not None:
        nx.set_node_attributes(G, {v: int(l) for v, l in enumerate(g.labels)}, "l")
    return G


def test_oracle_equals_networkx_vf2():
    """SPEC acceptance criterion 2 shape: G(30,0.2) and G(50,0.1),
    unlabeled and 3 labels, connected 3-5-node queries."""
    from networkx.algorithms import isomorphism as iso
    checked = 0
    for seed in range(1, 9):
        for (n, pn, pd) in [(30, 1, 5), (50, 1, 10)]:
            g = gi.random_gnp(n, pn, pd, seed)
            for nl in (0, 3):
                gg = g.with_labels(gi.uniform_labels(n, 3, seed + 7)) if nl else g
                q = gi.random_connected_query(3 + seed % 3, seed % 3, seed * 7 + n, nl)
                Gq = _nx(gi.from_edge_list(q.num_nodes, q.edges) if q.edges else gi.complete(1))
                if q.labels is not None:
                    import networkx as nx
                    nx.set_node_attributes(Gq, {v: l for v, l in enumerate(q.labels)}, "l")
                    gm = iso.GraphMatcher(_nx(gg), Gq, node_match=lambda a, b: a["l"] == b["l"])
                else:
                    gm = iso.GraphMatcher(_nx(gg), Gq)
                ref = {tuple(sorted(((v, u) for u, v in m.items()))) for m in gm.subgraph_monomorphisms_iter()}
                ref_rows = np.array(sorted(tuple(u for _, u in sorted(r)) for r in ref), dtype=np.int32).reshape(-1, q.num_nodes)
                cnt, rows = oracle.match(gg, q)
                assert cnt == len(ref_rows)
                np.testing.assert_array_equal(rows, oracle.sort_rows(ref_rows))
                checked += 1
    assert checked == 32


# ------------------------------------------------------------------ closed forms
@pytest.mark.parametrize("qname", ["K2", "K3", "P3", "P4", "S3", "C4", "K4", "C5", "house", "diamond"])
def test_complete_graph_closed_form(qname):
    q = gi.query(qname)
    for n in (5, 7):
        cnt, rows = oracle.match(gi.complete(n), q, count_only=False)
        assert cnt == cf.complete_graph(n, q.num_nodes)
        assert len({tuple(r) for r in rows.tolist()}) == cnt  # no duplicate rows


def test_labeled_complete_graph_closed_form():
    n = 9
    labels = np.array([0, 0, 0, 1, 1, 2, 2, 2, 2], np.uint32)
    g = gi.complete(n).with_labels(labels)
    counts = {0: 3, 1: 2, 2: 4}
    for qname, ql in [("K3", [0, 1, 2]), ("K3", [2, 2, 0]), ("P4", [1, 1, 2, 0]), ("S3", [2, 0, 0, 0]),
                      ("K4", [0, 0, 0, 0]), ("C4", [1, 2, 1, 2])]:
        q = gi.query(qname, ql)
        cnt, _ = oracle.match(g, q, count_only=True)
        assert cnt == cf.complete_graph_labeled(counts, ql), (qname, ql)


def test_star_closed_form_labeled():
    for seed in (1, 2, 3):
        g = gi.random_gnp(40, 1, 5, seed).with_labels(gi.uniform_labels(40, 3, seed))
        for ql in ([0, 1, 1, 2], [1, 2, 2, 2], [2, 0, 1, 2], [0, 0, 0, 0]):
            cnt, _ = oracle.match(g, gi.query("S3", ql), count_only=True)
            assert cnt == cf.star(g, ql[0], ql[1:]) == cf.star_vectorised(g, ql[0], ql[1:], 3)
    g = gi.random_gnp(40, 1, 5, 9)
    cnt, _ = oracle.match(g, gi.query("S3"), count_only=True)
    assert cnt == cf.star(g, 0, [0, 0, 0])


def test_path4_closed_form_labeled_and_unlabeled():
    for seed in (1, 2, 3):
        g = gi.random_gnp(40, 1, 5, seed).with_labels(gi.uniform_labels(40, 3, seed + 1))
        for ql in ([0, 1, 2, 0], [1, 2, 2, 1], [0, 0, 0, 0], [2, 1, 0, 1]):
            cnt, _ = oracle.match(g, gi.query("P4", ql), count_only=True)
            assert cnt == cf.path4_labeled(g, *ql) == cf.path4_labeled_vectorised(g, *ql, num_labels=3), ql
        gu = gi.random_gnp(40, 1, 5, seed)
        cnt, _ = oracle.match(gu, gi.query("P4"), count_only=True)
        assert cnt == cf.path4_unlabeled(gu, oracle.count_triangles(gu))


def test_cycle4_codegree_and_trace_forms():
    for seed in (1, 2):
        g = gi.random_gnp(30, 1, 4, seed)
        cnt, _ = oracle.match(g, gi.query("C4"), count_only=True)
        A = cf.dense_adj(g)
        assert cnt == cf.cycle4(g) == cf.cycle4_dense(A)
        cnt3, _ = oracle.match(g, gi.query("K3"), count_only=True)
        assert cnt3 == cf.triangle_trace(A)


def test_bipartite_petersen_grid_forms():
    for a, b in [(2, 3), (3, 4), (4, 4)]:
        g = gi.complete_bipartite(a, b)
        assert oracle.match(g, gi.query("C4"), count_only=True)[0] == cf.kab_c4(a, b)
        assert oracle.match(g, gi.query("K3"), count_only=True)[0] == 0
    p = gi.petersen()
    assert oracle.match(p, gi.query("C5"), count_only=True)[0] == 120
    assert oracle.match(p, gi.query("K3"), count_only=True)[0] == 0
    assert oracle.match(p, gi.query("C4"), count_only=True)[0] == 0
    for W, H in [(3, 4), (7, 5)]:
        assert oracle.match(gi.plain_grid(W, H), gi.query("C4"), count_only=True)[0] == cf.grid_plain_c4(W, H)
        assert oracle.match(gi.plain_grid(W, H), gi.query("K3"), count_only=True)[0] == 0


def test_grid_with_diagonals_clique_forms():
    g = gi.grid(40, 30, seed=5)
    d1, d2 = g.meta["d1"], g.meta["d2"]
    assert d2 > 0 and d1 > 0
    assert oracle.match(g, gi.query("K4"), count_only=True)[0] == cf.grid_diag_k4(d2)
    assert oracle.match(g, gi.query("K3"), count_only=True)[0] == cf.grid_diag_k3(d1, d2)
    assert oracle.match(g, gi.query("C4"), count_only=True)[0] == cf.cycle4(g)


# ------------------------------------------------------------------ symmetry
AUT_SIZES = {"K3": 6, "K4": 24, "P3": 2, "P4": 2, "C4": 8, "C5": 10, "S3": 6, "house": 2}


@pytest.mark.parametrize("qname,size", sorted(AUT_SIZES.items()))
def test_automorphism_group_sizes(qname, size):
    assert len(oracle.automorphisms(gi.query(qname))) == size


def test_labeled_automorphism_sizes():
    assert len(oracle.automorphisms(gi.query("P4", [0, 1, 1, 0]))) == 2
    assert len(oracle.automorphisms(gi.query("S3", [0, 1, 1, 2]))) == 2
    assert len(oracle.automorphisms(gi.query("S3", [0, 1, 1, 1]))) == 6
    assert len(oracle.automorphisms(gi.query("house", [0, 0, 1, 1, 2]))) == 2
    assert len(oracle.automorphisms(gi.query("house", [0, 1, 2, 3, 4]))) == 1


def test_orbit_identity_and_expansion():
    g = gi.random_gnp(25, 1, 3, 4)
    for qname in ["K3", "P4", "C4", "S3", "house", "K4"]:
        q = gi.query(qname)
        cnt, rows = oracle.match(g, q)
        aut = oracle.automorphisms(q)
        uniq = oracle.unique(rows, aut)
        assert len(aut) * len(uniq) == cnt
        np.testing.assert_array_equal(oracle.expand_orbits(uniq, aut), rows)


def test_label_sum_identity():
    """sum over all L^k labelings of Q of emb(Q_lambda, G) = emb(Q unlabeled, G)."""
    L = 2
    g = gi.random_gnp(20, 1, 3, 11).with_labels(gi.uniform_labels(20, L, 3))
    for qname in ["K3", "P4", "C4"]:
        q = gi.query(qname)
        total = sum(oracle.match(g, q.with_labels(list(lam)), count_only=True)[0]
                    for lam in itertools.product(range(L), repeat=q.num_nodes))
        assert total == oracle.match(g, q, count_only=True)[0]


# ------------------------------------------------------------------ exact counters
def test_clique_counters_against_dfs():
    for g in [gi.rmat(10, 8, seed=3), gi.grid(30, 30, seed=2), gi.random_gnp(60, 1, 4, 5), gi.complete(8)]:
        assert 6 * oracle.count_triangles(g) == oracle.match(g, gi.query("K3"), count_only=True)[0]
        assert 24 * oracle.count_k4(g) == oracle.match(g, gi.query("K4"), count_only=True)[0]
    assert oracle.count_triangles(gi.complete(9)) == 84
    assert oracle.count_k4(gi.complete(9)) == 126


def test_clique_counts_by_root_against_networkx():
    """Per-root clique counts (each clique counted at its lowest (degree, id)-ranked
    vertex) against networkx's clique enumeration — an implementation that shares
    nothing with the merge-based forward counter — and partition sums = totals."""
    import networkx as nx
    for g in [gi.rmat(9, 8, seed=4), gi.random_gnp(50, 1, 3, 9), gi.grid(12, 12, seed=3), gi.complete(7)]:
        rank = oracle.rank_order(g)
        deg = np.diff(g.offsets)
        # rank = position in sorted (deg, id) order, written out directly
        by = sorted(range(g.num_nodes), key=lambda v: (int(deg[v]), v))
        assert [int(rank[v]) for v in by] == list(range(g.num_nodes))
        G = _nx(g)
        for k in (3, 4):
            want = np.zeros(g.num_nodes, dtype=np.int64)
            for c in nx.enumerate_all_cliques(G):
                if len(c) == k:
                    want[min(c, key=lambda v: rank[v])] += 1
                elif len(c) > k:
                    break
            total, per = oracle.clique_counts_by_root(g, k)
            np.testing.assert_array_equal(per.astype(np.int64), want)
            assert total == int(want.sum()) == (oracle.count_triangles(g) if k == 3 else oracle.count_k4(g))
            sub = np.arange(1, g.num_nodes, 3, dtype=np.int32)
            t2, p2 = oracle.clique_counts_by_root(g, k, sub)
            np.testing.assert_array_equal(p2.astype(np.int64), want[sub])
            assert t2 == int(want[sub].sum())


def test_house_counter_against_dfs_and_brute_force():
    """The counting house oracle (roof x 4-path per edge) equals the DFS oracle's count,
    per root, on labeled graphs where every label condition holds, and brute force on tiny
    ones; patterns that would need explicit injectivity checks are refused."""
    cases = [(gi.rmat(10, 8, seed=5), 5, [0, 1, 2, 3, 4]), (gi.rmat(10, 8, seed=6), 3, [0, 0, 1, 1, 2]),
             (gi.random_gnp(80, 1, 4, 3), 4, [1, 0, 3, 2, 0]),  # l4 clash -> refused
             (gi.random_gnp(80, 1, 3, 4), 6, [2, 5, 1, 0, 3]), (gi.complete(9), 3, [0, 0, 1, 1, 2])]
    checked = 0
    for g0, L, labs in cases:
        g = g0.with_labels(gi.uniform_labels(g0.num_nodes, L, 7))
        if labs[4] in labs[:4]:
            with pytest.raises(ValueError):
                oracle.house_counts_by_root(g, labs)
            continue
        q = gi.query("house", labs)
        total, per = oracle.house_counts_by_root(g, labs)
        assert total == oracle.match(g, q, count_only=True)[0]
        roots = np.arange(0, g.num_nodes, 7, dtype=np.int32)
        t2, p2 = oracle.house_counts_by_root(g, labs, roots)
        assert t2 == oracle.match(g, q, roots=roots, count_only=True)[0]
        for v, c in zip(roots[:12], p2[:12]):
            assert c == oracle.match(g, q, roots=np.array([v], np.int32), count_only=True)[0]
        checked += 1
    assert checked >= 3
    for seed in range(6):  # brute force on tiny labeled graphs
        g = gi.random_gnp(8, 1, 2, 20 + seed).with_labels(gi.uniform_labels(8, 3, seed))
        labs = [0, 0, 1, 1, 2]
        assert oracle.house_counts_by_root(g, labs)[0] == len(oracle.brute_force(g, gi.query("house", labs)))
    with pytest.raises(ValueError):
        oracle.house_counts_by_root(gi.complete(6).with_labels(np.zeros(6, np.uint32)), [0, 1, 0, 1, 2])


@pytest.mark.parametrize("k,top", [(3, 1000), (4, 1 << 30), (2, -1)])
def test_sort_rows_against_python_sorted(k, top):
    """oracle.sort_rows = Python's sorted() on the rows as unsigned tuples (both of its
    branches: one packed 64-bit key when it fits, np.lexsort otherwise; negative int32
    values order as large unsigned ones)."""
    rng = np.random.default_rng(k)
    if top < 0:
        rows = rng.integers(-2**31, 2**31, size=(3000, k), dtype=np.int64).astype(np.int32)
    else:
        rows = rng.integers(0, top, size=(3000, k)).astype(np.int32)
    rows[100:200] = rows[0:100]  # ties
    got = oracle.sort_rows(rows)
    want = sorted((tuple(int(x) & 0xffffffff for x in r) for r in rows))
    assert [tuple(int(x) & 0xffffffff for x in r) for r in got] == want


# ------------------------------------------------------------------ restriction / invariance
def test_root_subset_partition_union():
    g = gi.rmat(9, 8, seed=2).with_labels(gi.uniform_labels(512, 2, 2))
    q = gi.query("P4", [0, 1, 1, 0])
    cnt, rows = oracle.match(g, q)
    parts = [np.arange(s, 512, 3, dtype=np.int32) for s in range(3)]
    sub = [oracle.match(g, q, roots=p) for p in parts]
    assert sum(c for c, _ in sub) == cnt
    np.testing.assert_array_equal(oracle.sort_rows(np.concatenate([r for _, r in sub])), rows)
    for p, (_, r) in zip(parts, sub):
        assert np.isin(r[:, 0], p).all()


def test_relabel_invariance():
    g = gi.random_gnp(30, 1, 4, 6)
    perm = np.random.default_rng(0).permutation(30)
    src = np.repeat(np.arange(30), np.diff(g.offsets))
    g2 = gi.csr_from_edges(30, perm[src], perm[g.cols])
    for qname in ["K3", "C4", "P4"]:
        _, r1 = oracle.match(g, gi.query(qname))
        _, r2 = oracle.match(g2, gi.query(qname))
        np.testing.assert_array_equal(oracle.sort_rows(perm[r1].astype(np.int32)), r2)


def test_oracle_rejects_bad_queries():
    g = gi.complete(4)
    with pytest.raises(ValueError):
        oracle.match(g, gi.Query(3, [(0, 1)], None))  # disconnected
    with pytest.raises(ValueError):
        oracle.match(g, gi.query("K3", [0, 0, 0]))  # query labels, no data labels
