"""Host plan (Alg. 1 PreCompute_on_CPUs) through
the C ABI's host-only gsm_plan_query — no GPU needed (marked not-gpu).
Pinned against brute-force Aut(Q) from the oracle package and against the
orbit property of the ID constraints (SURVEY §8(c) amb. 9, "Host plan" pin)."""
import itertools

import numpy as np
import pytest

import gsm_inputs as gi
import oracle
from paper_2003_01527_b200 import gsm


def plan(q, cand=None, flags=0):
    return gsm.gsm_plan_query(q.num_nodes, q.edges, q.labels, cand, flags)


EXPECTED_CONDITIONS = {
    ("K3", None): {(0, 1), (0, 2), (1, 2)},
    ("P3", None): {(0, 2)},
    ("P4", None): {(0, 3)},
    ("C4", None): {(0, 1), (0, 2), (0, 3), (1, 3)},
    ("K4", None): {(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)},
    ("S3", None): {(1, 2), (1, 3), (2, 3)},
    ("house", None): {(0, 1)},
    ("P4", (0, 1, 1, 0)): {(0, 3)},
    ("S3", (0, 1, 1, 2)): {(1, 2)},
    ("house", (0, 1, 2, 3, 4)): set(),
}


@pytest.mark.parametrize("key", sorted(EXPECTED_CONDITIONS, key=str))
def test_grochow_kellis_conditions(key):
    name, labels = key
    p = plan(gi.query(name, None if labels is None else list(labels)))
    assert set(map(tuple, p["conditions"])) == EXPECTED_CONDITIONS[key]


def _random_queries():
    out = []
    for seed in range(40):
        k = 3 + seed % 5
        out.append(gi.random_connected_query(k, seed % 4, 1000 + seed, 0))
        out.append(gi.random_connected_query(k, seed % 4, 2000 + seed, 2))
    for name in gi.QUERIES:
        out.append(gi.query(name))
    return out


def test_automorphism_order_matches_brute_force():
    for q in _random_queries():
        assert plan(q)["automorphisms"] == len(oracle.automorphisms(q)), q.name


def test_conditions_pick_exactly_one_per_orbit():
    """For every embedding list, exactly one member of each Aut(Q) orbit satisfies
    the constraints, for two different strict total orders on data vertices."""
    g = gi.random_gnp(14, 1, 2, 3).with_labels(gi.uniform_labels(14, 2, 1))
    deg = np.diff(g.offsets)
    orders = {"id": np.arange(14), "deg,id": np.lexsort((np.arange(14), deg)).argsort()}
    checked = 0
    for q in _random_queries():
        if q.num_nodes > 6:
            continue
        _, rows = oracle.match(g, q)
        if len(rows) == 0:
            continue
        aut = oracle.automorphisms(q)
        conds = plan(q)["conditions"]
        canon = oracle.canonical(rows, aut)
        for name, rank in orders.items():
            ok = np.ones(len(rows), bool)
            for a, b in conds:
                ok &= rank[rows[:, a]] < rank[rows[:, b]]
            sel = canon[ok]
            # one member per orbit: the selected rows' canonical forms are all distinct and cover all orbits
            assert len(sel) == len(oracle.unique(rows, aut)), (q.name, name)
            assert len({tuple(r) for r in sel.tolist()}) == len(sel)
            checked += 1
    assert checked > 20


def test_order_invariants_and_priorities():
    for q in _random_queries():
        k = q.num_nodes
        E = {frozenset(e) for e in q.edges}
        cand = [(7 * u + 3) % 5 + 1 for u in range(k)]
        p = plan(q, cand)
        order = p["order"]
        assert sorted(order) == list(range(k))
        qdeg = [sum(1 for e in q.edges if u in e) for u in range(k)]
        # first vertex: min |C(u)|, then max degree, then min id
        best = min(range(k), key=lambda u: (cand[u], -qdeg[u], u))
        assert order[0] == best
        rebuilt = set()
        for i in range(1, k):
            back = [j for j in range(i) if frozenset((order[i], order[j])) in E]
            assert back, "every later position has a backward neighbour (connected prefix)"
            assert p["parent"][i] == back[0]
            assert p["backward"][i] == sum(1 << j for j in back)
            rebuilt |= {frozenset((order[i], order[j])) for j in back}
            # greedy rule: max d_M among the remaining, then min |C|, max deg, min id
            placed = set(order[:i])
            rem = [u for u in range(k) if u not in placed]
            dm = {u: sum(1 for w in placed if frozenset((u, w)) in E) for u in rem}
            exp = min(rem, key=lambda u: (-dm[u], cand[u], -qdeg[u], u))
            assert order[i] == exp
        assert rebuilt == E  # parents + non-tree edges = E_Q


def test_no_symmetry_flag_drops_conditions():
    p = plan(gi.query("K4"), flags=gsm.GSM_FLAG_NO_SYMMETRY)
    assert p["conditions"] == [] and p["automorphisms"] == 24


@pytest.mark.parametrize("k,edges", [(3, [(0, 1)]), (3, [(0, 1), (0, 1), (1, 2)]), (3, [(0, 0), (0, 1), (1, 2)]),
                                     (0, []), (33, [(i, i + 1) for i in range(32)]), (3, [(0, 5), (1, 2)])])
def test_invalid_queries(k, edges):
    with pytest.raises(gsm.GsmError) as e:
        gsm.gsm_plan_query(k, edges)
    assert e.value.status == 3


def test_large_symmetric_query_group_order():
    # K_8: |Aut| = 8! without listing; star K_{1,7}: 7!
    assert gsm.gsm_plan_query(8, list(itertools.combinations(range(8), 2)))["automorphisms"] == 40320
    assert gsm.gsm_plan_query(8, [(0, i) for i in range(1, 8)])["automorphisms"] == 5040


def _pair_expected(q, conds):
    """Brute force: does Q have non-adjacent a, b with no condition between them and
    Q - {a, b} connected?  (the pair-tail eligibility)"""
    k = q.num_nodes
    adj = {u: set() for u in range(k)}
    for a, b in q.edges:
        adj[a].add(b)
        adj[b].add(a)
    for a in range(k):
        for b in range(a + 1, k):
            if b in adj[a] or (a, b) in conds or (b, a) in conds:
                continue
            rest = [u for u in range(k) if u not in (a, b)]
            seen, stack = {rest[0]}, [rest[0]]
            while stack:
                x = stack.pop()
                for y in adj[x]:
                    if y in rest and y not in seen:
                        seen.add(y)
                        stack.append(y)
            if len(seen) == len(rest):
                return True
    return False


@pytest.mark.parametrize("key", ["P3", "P4", "S3", "C4", "K4", "house", "tailed_triangle", "diamond", "K3"])
@pytest.mark.parametrize("labels", [None, "distinct"])
def test_count_mode_pair_tail_order(key, labels):
    """GSM_FLAG_PLAN_COUNT: when Q allows it the last two positions are non-adjacent, carry no
    ID condition between them, and every earlier position keeps a connected prefix; else the
    order is the plain greedy one (cliques, C4 with its conditions)."""
    q0 = gi.query(key)
    q = q0 if labels is None else gi.query(key, list(range(q0.num_nodes)))
    base = plan(q)
    p = plan(q, flags=gsm.GSM_FLAG_PLAN_COUNT)
    conds = set(p["conditions"])
    assert sorted(p["order"]) == list(range(q.num_nodes))
    for i in range(1, q.num_nodes):  # connected prefix at every position
        assert p["backward"][i] != 0, (key, p)
    a, b = p["order"][-2], p["order"][-1]
    adjacent = any({a, b} == {x, y} for x, y in q.edges)
    if _pair_expected(q, conds):
        assert not adjacent and (a, b) not in conds and (b, a) not in conds, (key, p)
        assert not (p["backward"][-1] >> (q.num_nodes - 2)) & 1
    else:
        assert p["order"] == base["order"], (key, p, base)
