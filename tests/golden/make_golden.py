"""Generate the golden vectors that pin the oracle (and the GPU path) to the
reference implementation itself.

Run in the build container, where the reference is importable:
    python tests/golden/make_golden.py [/root/reference/pkg/src]
It imports `giftplace` from the reference checkout (read-only), evaluates the
hot path on fixed inputs and writes tests/golden/golden.npz plus
tests/golden/golden_meta.json (library versions, hashes).  Nothing here runs
on the GPU box: the reference does not travel; only these fixtures do.

Cases
  kat_*      the reference's own KAT inputs (test_graph.py / test_gift.py)
  rand_*     random_connected_graph-style COO graphs (conftest.py:62-82 recipe),
             plus raw COO with duplicates, negative values and cancellations
  dupnets    a small netlist whose nets repeat cells and mix pin counts, so
             duplicate keys with >= 3 unequal 2/m contributions exist (the
             introsort-order-sensitive case)
  adversary  one COO row whose columns are McIlroy killer keys for libstdc++
             introsort (heapsort fallback) with unequal duplicate values
  c0         BASELINE config 0 (synth.generate('c0', seed=1)): full CSR /
             degree / placement hashes and sampled rows
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
REF_SRC = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import giftplace as gp  # noqa: E402  (the reference)
import scipy  # noqa: E402

from oracle import oracle as orc  # noqa: E402  (only for the adversarial keys generator)
from paper_2502_17632_b200 import synth  # noqa: E402


def h(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_design(n_cells, nets_pins, fixed=None, region=(0.0, 0.0, 10.0, 10.0)):
    fixed = fixed or {}
    cells = []
    for i in range(n_cells):
        if i in fixed:
            cells.append(gp.Cell(id=i, name=f"c{i}", width=1.0, height=1.0, fixed=True, fixed_pos=fixed[i]))
        else:
            cells.append(gp.Cell(id=i, name=f"c{i}", width=1.0, height=1.0))
    nets = [gp.Net(id=j, name=f"n{j}", pins=[gp.Pin(int(c)) for c in p]) for j, p in enumerate(nets_pins)]
    d = gp.Design(cells=cells, nets=nets, region=gp.Region(*region))
    d.validate()
    return d


def flat(nets_pins):
    counts = np.array([len(p) for p in nets_pins], dtype=np.int64)
    ns = np.zeros(len(nets_pins) + 1, dtype=np.int64)
    np.cumsum(counts, out=ns[1:])
    pc = np.array([c for p in nets_pins for c in p], dtype=np.int64)
    return ns, pc


def random_graph_coo(n, rng):
    """conftest.py:62-82 recipe (spanning tree + n/2 extra edges, both triangles)."""
    rows, cols, vals = [], [], []
    order = rng.permutation(n)
    for i in range(1, n):
        a = order[i]
        b = order[rng.integers(0, i)]
        rows += [a, b]
        cols += [b, a]
        w = float(rng.uniform(0.1, 2.0))
        vals += [w, w]
    for _ in range(max(n // 2, 1)):
        a, b = rng.integers(0, n, size=2)
        if a == b:
            continue
        w = float(rng.uniform(0.1, 2.0))
        rows += [int(a), int(b)]
        cols += [int(b), int(a)]
        vals += [w, w]
    return np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64), np.array(vals, dtype=np.float64)


def main() -> None:
    out: dict[str, np.ndarray] = {}
    meta = {"numpy": np.__version__, "scipy": scipy.__version__, "reference": REF_SRC, "cases": {}}

    def put_csr(name, adj):
        out[f"{name}__indptr"] = np.asarray(adj.indptr, dtype=np.int64)
        out[f"{name}__indices"] = np.asarray(adj.indices, dtype=np.int64)
        out[f"{name}__values"] = np.asarray(adj.values, dtype=np.float64)
        out[f"{name}__degrees"] = np.asarray(adj.degrees, dtype=np.float64)

    # ---- netlist KATs (test_graph.py:51-103, test_gift.py) ----
    kats = {
        "kat_two_pin": (2, [[0, 1]]),
        "kat_three_pin": (3, [[0, 1, 2]]),
        "kat_parallel": (2, [[0, 1], [0, 1]]),
        "kat_degenerate": (3, [[0], [], [1, 2]]),
        "kat_self_pairs": (2, [[0, 0, 1]]),
        "kat_cap": (5, [[0, 1, 2, 3, 4], [0, 1]]),
        "kat_tri": (3, [[0, 1, 2], [0, 1]]),
    }
    rng = np.random.default_rng(20240817)
    nets = [list(rng.choice(30, size=rng.integers(2, 6), replace=True)) for _ in range(40)]
    kats["kat_brute"] = (30, [[int(c) for c in net] for net in nets])
    # duplicate-heavy netlist: mixed pin counts on a small cell set
    r2 = np.random.default_rng(7)
    dn = []
    for _ in range(3000):
        m = int(r2.choice([2, 3, 4, 5, 7, 9, 13, 21]))
        dn.append([int(c) for c in r2.integers(0, 60, size=m)])
    kats["dupnets"] = (60, dn)
    for name, (n, np_) in kats.items():
        d = ref_design(n, np_)
        cap = 3 if name == "kat_cap" else None
        adj = gp.build_clique_graph(d, max_clique_pins=cap)
        ns, pc = flat(np_)
        out[f"{name}__net_start"] = ns
        out[f"{name}__pin_cell"] = pc
        out[f"{name}__n"] = np.array([n, -1 if cap is None else cap], dtype=np.int64)
        put_csr(name, adj)
        for sigma in (0.0, 1.0, 2.0, 4.0):
            try:
                op = gp.normalized_augmented_adjacency(adj, sigma)
                out[f"{name}__norm{sigma:g}__indptr"] = np.asarray(op.indptr, dtype=np.int64)
                out[f"{name}__norm{sigma:g}__indices"] = np.asarray(op.indices, dtype=np.int64)
                out[f"{name}__norm{sigma:g}__values"] = np.asarray(op.values, dtype=np.float64)
            except gp.IsolatedNodeError as e:
                out[f"{name}__norm{sigma:g}__isolated"] = np.array([e.node], dtype=np.int64)
        g = np.random.default_rng(3).standard_normal((n, 2)) * 10.0
        out[f"{name}__g"] = g
        try:
            out[f"{name}__filter"] = gp.gift_filter(adj, g)
        except gp.IsolatedNodeError:
            pass
        meta["cases"][name] = {"n": n, "nets": len(np_), "nnz": int(adj.nnz)}

    # ---- COO cases (from_coo, graph.py:114-117) ----
    rng = np.random.default_rng(812)
    for i, n in enumerate((15, 60, 150)):
        r, c, v = random_graph_coo(n, rng)
        adj = gp.from_coo(n, r, c, v)
        name = f"rand_graph{i}"
        out[f"{name}__coo"] = np.stack([r.astype(np.float64), c.astype(np.float64), v])
        out[f"{name}__n"] = np.array([n], dtype=np.int64)
        put_csr(name, adj)
        g = rng.standard_normal((n, 2)) * 10.0
        out[f"{name}__g"] = g
        out[f"{name}__filter"] = gp.gift_filter(adj, g)
        terms = (gp.FilterTerm(sigma=1.0, k=1, alpha=0.5), gp.FilterTerm(sigma=1.0, k=3, alpha=0.5))
        out[f"{name}__filter_custom"] = gp.gift_filter(adj, g, gp.GiftConfig(terms=terms))
        op = gp.normalized_augmented_adjacency(adj, 4.0)
        out[f"{name}__pow3"] = gp.apply_operator_power(op, g, 3)
        meta["cases"][name] = {"n": n, "nnz": int(adj.nnz)}
    # raw symmetric COO with duplicates, negative values and exact cancellations
    for i in range(3):
        n = 40
        k = 900
        r = rng.integers(0, n, k)
        c = rng.integers(0, n, k)
        v = rng.standard_normal(k)
        v[: k // 10] = 0.0
        rr = np.concatenate([r, c, r[:50]])
        cc = np.concatenate([c, r, c[:50]])
        vv = np.concatenate([v, v, np.zeros(50)])
        name = f"rand_coo{i}"
        # mirror the cancellations on both triangles
        rr = np.concatenate([rr, r[50:60], c[50:60]])
        cc = np.concatenate([cc, c[50:60], r[50:60]])
        vv = np.concatenate([vv, -v[50:60], -v[50:60]])
        adj = gp.from_coo(n, rr, cc, vv)
        out[f"{name}__coo"] = np.stack([rr.astype(np.float64), cc.astype(np.float64), vv])
        out[f"{name}__n"] = np.array([n], dtype=np.int64)
        put_csr(name, adj)
        meta["cases"][name] = {"n": n, "nnz": int(adj.nnz)}
    # adversarial introsort row (heapsort fallback) with unequal duplicates
    # McIlroy keys //4: four-fold duplicate columns, still drives introsort into
    # its heapsort fallback (checked with oracle.heapsort_calls())
    keys = orc.antiqsort_keys(1500) // 4
    n = int(keys.max()) + 2
    r0 = n - 1  # the adversarial row's own index is not among its columns
    row = np.full(len(keys), r0, dtype=np.int64)
    vals = np.random.default_rng(5).standard_normal(len(keys))
    rr = np.concatenate([row, keys])
    cc = np.concatenate([keys, row])
    vv = np.concatenate([vals, vals])
    import scipy.sparse as sp

    up = sp.coo_matrix((vv, (rr, cc)), shape=(n, n)).tocsr()
    out["adversary__coo"] = np.stack([rr.astype(np.float64), cc.astype(np.float64), vv])
    out["adversary__n"] = np.array([n], dtype=np.int64)
    out["adversary__indptr"] = up.indptr.astype(np.int64)
    out["adversary__indices"] = up.indices.astype(np.int64)
    out["adversary__values"] = up.data.astype(np.float64)
    meta["cases"]["adversary"] = {"n": n, "nnz": int(up.nnz)}

    # ---- metrics consumers (§8(f)): laplacian (exact), S, R, HPWL ----
    for name in ("kat_brute", "dupnets", "rand_graph1"):
        if name.startswith("rand"):
            coo = out[f"{name}__coo"]
            adj = gp.from_coo(int(out[f"{name}__n"][0]), coo[0].astype(np.int64), coo[1].astype(np.int64), coo[2])
        else:
            n_ = int(out[f"{name}__n"][0])
            adj = gp.build_clique_graph(ref_design(n_, [list(map(int, out[f"{name}__pin_cell"][a:b]))
                                                        for a, b in zip(out[f"{name}__net_start"][:-1],
                                                                        out[f"{name}__net_start"][1:])]))
        lap = gp.laplacian(adj)
        out[f"{name}__lap__indptr"] = np.asarray(lap.indptr, dtype=np.int64)
        out[f"{name}__lap__indices"] = np.asarray(lap.indices, dtype=np.int64)
        out[f"{name}__lap__values"] = np.asarray(lap.values, dtype=np.float64)
        g = out[f"{name}__g"]
        out[f"{name}__qwl"] = np.array([gp.quadratic_wirelength(adj, g)])
        out[f"{name}__rayleigh"] = np.array([gp.rayleigh_smoothness(lap, g[:, 0]),
                                             gp.rayleigh_smoothness(lap, g[:, 1], center=False)])

    # ---- BASELINE config 0 ----
    fd = synth.generate("c0", seed=1)
    d = fd.to_design(gp)
    adj = gp.build_clique_graph(d, max_clique_pins=fd.meta["max_clique_pins"])
    cfg = gp.GiftConfig(seed=0, jitter_scale=10.0)
    g0 = gp.initial_signal(d, cfg)
    g32 = g0.astype(np.float32).astype(np.float64)
    filt = gp.gift_filter(adj, g32)
    placed, _ = gp.gift_place(d, adj, cfg)
    ind = np.asarray(adj.indices, dtype=np.int64)
    c0 = {
        "n": int(adj.n), "nnz": int(adj.nnz),
        "indptr_sha": h(np.asarray(adj.indptr, dtype=np.int64)),
        "indices_sha": h(ind),
        "values_sha": h(np.asarray(adj.values, dtype=np.float64)),
        "degrees_sha": h(np.asarray(adj.degrees, dtype=np.float64)),
        "g0_sha": h(g0), "filter_g32_sha": h(filt), "place_sha": h(placed),
    }
    meta["cases"]["c0"] = c0
    out["c0__qwl"] = np.array([gp.quadratic_wirelength(adj, g0), gp.quadratic_wirelength(adj, placed)])
    out["c0__hpwl"] = np.array([gp.hpwl(d, g0), gp.hpwl(d, placed)])
    lap0 = gp.laplacian(adj)
    out["c0__rayleigh"] = np.array([gp.rayleigh_smoothness(lap0, placed[:, 0]),
                                    gp.rayleigh_smoothness(lap0, placed[:, 1])])
    sample = np.arange(0, adj.n, 97)
    out["c0__sample_rows"] = sample
    out["c0__degrees_sample"] = np.asarray(adj.degrees)[sample]
    out["c0__filter_g32_sample"] = filt[sample]
    out["c0__place_sample"] = placed[sample]

    # ---- .pl writer (§8(f) row 4): the reference's write_placement bytes ----
    import tempfile
    rng = np.random.default_rng(20261020)
    edge_cx = [0.5078125, 1e22, -1e-9 + 0.5, 2.5e-6 + 0.5, float("nan"), float("inf"), -float("inf"), 5e-324,
               123456789.1234565, 1e15 + 0.5, -0.0, 0.5, -2.5, 0.0000005 + 0.5, 1.0000005, 999999.9999995]
    n_pl = 64
    cells = []
    for i in range(n_pl):
        w = [1.0, 2.0, 3.0, 0.5, 1e-3, 0.0][i % 6]
        name = ["c%d" % i, "cell_%03d" % i, "u\u00e9%d" % i, "x/y[%d]" % i][i % 4]
        fixed = i % 5 == 0
        cells.append(gp.Cell(id=i, name=name, width=w, height=[1.0, 2.0, 0.25][i % 3], fixed=fixed,
                             fixed_pos=(0.0, 0.0) if fixed else None))
    pl = rng.normal(0.0, 1e4, size=(n_pl, 2))
    pl[: len(edge_cx), 0] = edge_cx
    pl[: len(edge_cx), 1] = edge_cx[::-1]
    pl[20:30] = np.round(pl[20:30], 7) + 5e-7  # near-ties at the 6th decimal
    pl[17] = (-0.0, 0.0078125)   # width 0: "-0.000000", an exact tie (to even)
    pl[35] = (-1e-9, -4e-7)      # negatives that round to "-0.000000"
    pl[41] = (2.0 ** 100, -(2.0 ** 90) - 0.0)  # wide integer parts (exact %.6f of large binaries)
    dpl = gp.Design(cells=cells, nets=[], region=gp.Region(0.0, 0.0, 10.0, 10.0))
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "edge.pl")
        gp.write_placement(dpl, pl, path)
        text = open(path, "rb").read()
        out["pl_edge__pos"] = pl
        out["pl_edge__width"] = np.array([c.width for c in cells])
        out["pl_edge__height"] = np.array([c.height for c in cells])
        out["pl_edge__fixed"] = np.array([c.fixed for c in cells], dtype=np.uint8)
        out["pl_edge__names"] = np.frombuffer("\n".join(c.name for c in cells).encode(), dtype=np.uint8)
        out["pl_edge__text"] = np.frombuffer(text, dtype=np.uint8)
        path = os.path.join(td, "c0.pl")
        gp.write_placement(d, placed, path)
        text = open(path, "rb").read()
        meta["cases"]["pl_c0"] = {"bytes": len(text), "sha": hashlib.sha256(text).hexdigest()}
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    with open(os.path.join(HERE, "golden_meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print(f"wrote {len(out)} arrays; c0 nnz {adj.nnz}")


if __name__ == "__main__":
    main()
