"""Pins of the oracle to values the paper prints (worked examples) -- no GPU needed.

Each fixture under tests/golden/ carries its PAPER.md citation.
"""
import numpy as np
import pytest

import oracle as O
import workloads as W


def _fig2_ops(g):
    N = g["N"]
    return [W.from_coo([0] * len(v), v, [1.0] * len(v), 1, N) for v in (g["vectors"][n] for n in "abc")]


def _fig3_ops(g):
    M, N = g["shape"]
    return [W.from_coo([r for r, _ in g[n]], [c for _, c in g[n]], np.arange(1, 13, dtype=np.float32), M, N)
            for n in ("A", "B")]


@pytest.mark.parametrize("method", ["rank", "alg1"])
def test_fig2_three_vector_partition(golden, method):
    g = golden("fig2_vec_lb.json")
    ops = _fig2_ops(g)
    parts = O.partition_rank(ops, g["P"]) if method == "rank" else O.partition_alg1(ops, g["P"])
    assert [[int(r), int(c)] for r, c in zip(parts.row, parts.col)] == g["boundaries_row_col"]
    assert parts.pos2().tolist() == g["boundary_positions_abc"]
    # cut points in the 1-D coordinate space of the figure: [0,2) [2,5) [5,10) [10,12)
    cuts = [int(c) if int(r) == 0 else g["N"] for r, c in zip(parts.row, parts.col)]
    assert cuts == g["cuts_coordinate_space"]
    work = np.diff(parts.pos2().sum(axis=1))
    assert work.tolist() == g["nnz_per_partition"]


def test_fig2_union_counts(golden):
    g = golden("fig2_vec_lb.json")
    ops = _fig2_ops(g)
    parts = O.partition_rank(ops, g["P"])
    assert O.spadd_counts(ops, parts).tolist() == g["union_counts_per_partition"]
    z_pos, z_crd, _ = O.spadd_k(ops)
    assert z_crd.tolist() == g["union"]


@pytest.mark.parametrize("method", ["rank", "alg1"])
def test_fig3a_dcsr_add_partition(golden, method):
    g = golden("fig3a_dcsr_add.json")
    ops = _fig3_ops(g)
    assert ops[0].pos.tolist() == g["A_pos"] and ops[1].pos.tolist() == g["B_pos"]
    parts = O.partition_rank(ops, g["P"]) if method == "rank" else O.partition_alg1(ops, g["P"])
    assert [[int(r), int(c)] for r, c in zip(parts.row, parts.col)] == g["boundaries_row_col"]
    assert parts.pos2().tolist() == g["boundary_positions_AB"]
    assert np.diff(parts.pos2().sum(axis=1)).tolist() == g["work_per_partition"]
    # the figure's colours: entry q of operand o belongs to partition p iff pos_p[o] <= q < pos_{p+1}[o]
    pos = parts.pos2()
    for o, key in enumerate(("A_partition_colour_index", "B_partition_colour_index")):
        member = [int(np.searchsorted(pos[:, o], q, side="right") - 1) for q in range(12)]
        assert member == g[key]


def test_fig3a_spadd_structure(golden):
    g = golden("fig3a_dcsr_add.json")
    ops = _fig3_ops(g)
    parts = O.partition_rank(ops, g["P"])
    cnt = O.spadd_counts(ops, parts)
    assert cnt.tolist() == g["spadd_counts"]
    assert np.concatenate([[0], np.cumsum(cnt)]).tolist() == g["spadd_offsets"]
    z_pos, z_crd, z_val = O.spadd_k(ops)
    assert z_pos.tolist() == g["Z_pos"] and len(z_crd) == g["nnz_Z"]
    # Z.pos[i+1] writer: the partition p with b_p.row <= i < b_{p+1}.row (Listing 8 guard, R7/I8)
    writers = [int(np.searchsorted(parts.row, i, side="right") - 1) for i in range(g["shape"][0])]
    assert writers == g["Z_pos_writer_partition_by_row"]


def test_listing5_and_lb_search(golden):
    g = golden("listing5_costs.json")
    pos = np.array(g["A_pos"])
    for x, c in g["C_i"].items():
        assert int(pos[int(x)] - pos[0]) == c
    cb = g["count_below"]
    assert O.lb_search(cb["crd"], cb["lo"], cb["hi"], cb["x"]) - cb["lo"] == cb["expect"]
    f2 = golden("fig2_vec_lb.json")["vectors"]
    total = sum(O.lb_search(v, 0, len(v) - 1, 5) for v in f2.values())
    assert total == g["fig2_dim_cost_x5"]["expect"]
