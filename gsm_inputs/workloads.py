"""The BASELINE.json configs as concrete, seeded workloads.

Each workload = one data graph (+ labels) and the list of queries one bench
"step" runs.  Shared by tests and bench.py; contains no method arithmetic."""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import gsm_inputs as gi


@dataclasses.dataclass
class Workload:
    name: str
    config_index: int
    description: str
    graph_fn: object
    queries: List[gi.Query]
    num_labels: int = 0
    label_seed: int = 1
    mem_budget_bytes: int = 0

    def graph(self) -> gi.Graph:
        g = self.graph_fn()
        if self.num_labels:
            g = g.with_labels(gi.uniform_labels(g.num_nodes, self.num_labels, self.label_seed),
                              tag=f"-L{self.num_labels}")
        return g


def _er(seed):
    return lambda: gi.erdos_renyi(1000, 4000, seed)


WORKLOADS = {
    # configs[0]: unlabeled triangle on G(1000, 4000), seeds 1..3 (seed 1 here)
    "er1000": Workload("er1000", 0, "G(n=1000,m=4000) unlabeled K3", _er(1), [gi.query("K3")]),
    # configs[1]: R-MAT scale 16, ef 16, 8 uniform labels; labeled P4 and star queries
    "rmat16": Workload("rmat16", 1, "R-MAT-16 ef16, 8 labels; P4 (0,1,2,3),(1,2,2,1); S3 (0;1,1,2),(0;1,2,3)",
                       lambda: gi.rmat(16, 16, 1),
                       [gi.query("P4", [0, 1, 2, 3]), gi.query("P4", [1, 2, 2, 1]),
                        gi.query("S3", [0, 1, 1, 2]), gi.query("S3", [0, 1, 2, 3])], num_labels=8),
    # configs[2]: 1000x1000 road-like grid with random diagonals; C4 and K4
    "grid1m": Workload("grid1m", 2, "1000x1000 grid + diagonals; C4, K4", lambda: gi.grid(1000, 1000, 1),
                       [gi.query("C4"), gi.query("K4")]),
    # configs[3]: R-MAT scale 22, 16 labels; labeled house (2 non-tree edges)
    "rmat22": Workload("rmat22", 3, "R-MAT-22 ef16, 16 labels; house (0,1,2,3,4),(0,0,1,1,2)",
                       lambda: gi.rmat(22, 16, 1),
                       [gi.query("house", [0, 1, 2, 3, 4]), gi.query("house", [0, 0, 1, 1, 2])], num_labels=16),
    # configs[4]: R-MAT scale 24, unlabeled; K3 and K4 with a fixed budget forcing chunking
    "rmat24": Workload("rmat24", 4, "R-MAT-24 ef16 unlabeled; K3, K4 (16 GiB frontier budget)",
                       lambda: gi.rmat(24, 16, 1), [gi.query("K3"), gi.query("K4")],
                       mem_budget_bytes=16 << 30),
    # development workloads (not BASELINE configs)
    "rmat20": Workload("rmat20", -1, "R-MAT-20 ef16 unlabeled; K3, K4", lambda: gi.rmat(20, 16, 1),
                       [gi.query("K3"), gi.query("K4")], mem_budget_bytes=4 << 30),
    "rmat24_k3": Workload("rmat24_k3", 4, "R-MAT-24 ef16 unlabeled; K3 only", lambda: gi.rmat(24, 16, 1),
                          [gi.query("K3")], mem_budget_bytes=16 << 30),
}


def get(name: str) -> Workload:
    return WORKLOADS[name]
