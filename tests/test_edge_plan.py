"""Host logic of the shared-edge blocks (csrc/edges.cu, gk_edge_blocks_plan):
no device needed.

Every triangle sits at exactly one block position; a block's triangles that
share a mesh edge (the same unordered vertex pair) share its block-local
index, distinct edges get distinct indices, and a block never exceeds
32 * chunks distinct edges.  These are the facts the combine step
Z[p][q] = E[e0(q)] + E[e1(q)] + E[e2(q)] relies on.
"""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def gk():
    import paper_1901_04162_b200 as g
    return g


def _check_plan(mesh, plan, chunks):
    tris = mesh.triangles
    nt = tris.shape[0]
    order, eidx = plan["order"], plan["edge_index"]
    start, nedge = plan["block_start"], plan["block_edges"]
    assert np.array_equal(np.sort(order), np.arange(nt))          # a permutation
    assert start[0] == 0 and start[-1] == nt and np.all(np.diff(start) > 0)
    assert np.all(nedge <= 32 * chunks)
    for b in range(len(nedge)):
        seen = {}
        for j in range(start[b], start[b + 1]):
            t = tris[order[j]]
            for s in range(3):
                key = tuple(sorted((int(t[s]), int(t[(s + 1) % 3]))))
                idx = int(eidx[j, s])
                assert idx < nedge[b]
                assert seen.setdefault(key, idx) == idx                # shared edge, one index
        assert len(seen) == nedge[b]                                   # distinct edges, distinct indices
        assert sorted(seen.values()) == list(range(nedge[b]))


@pytest.mark.parametrize("chunks", [1, 4, 11])
def test_sphere_blocks(gk, chunks):
    mesh = gk.jitter(gk.generate_sphere_mesh(1.0, 3), 1901, 1e-3)
    plan = gk.edge_blocks_plan(mesh, chunks)
    _check_plan(mesh, plan, chunks)
    # a closed mesh: about 1.5 distinct edges per triangle, plus block boundaries
    ratio = plan["block_edges"].sum() / (3.0 * mesh.triangle_count())
    assert 0.5 < ratio < (0.62 if chunks == 11 else 0.8)


@pytest.mark.parametrize("order_mode", [-1, 0, 1])
def test_plate_blocks_and_order(gk, order_mode):
    """the row-major plate: the bisection order is chosen (compact blocks)"""
    mesh = gk.generate_plate_mesh(1.0, 30)
    plan = gk.edge_blocks_plan(mesh, 4, order_mode)
    _check_plan(mesh, plan, 4)
    assert plan["ordered"] == (order_mode != 0)
    if order_mode == 0:
        assert np.array_equal(plan["order"], np.arange(mesh.triangle_count()))


def test_disconnected_triangles(gk):
    """no shared edges: three per triangle, blocks of at most 32 chunks / 3"""
    rng = np.random.default_rng(7)
    N = 100
    verts = (rng.uniform(-1, 1, (N, 1, 3)) + rng.uniform(-0.05, 0.05, (N, 3, 3))).reshape(-1, 3)
    mesh = gk.TriangleMesh(verts, np.arange(3 * N, dtype=np.uint32).reshape(N, 3))
    plan = gk.edge_blocks_plan(mesh, 1, 0)
    _check_plan(mesh, plan, 1)
    assert plan["block_edges"].sum() == 3 * N and np.all(np.diff(plan["block_start"]) <= 10)


def test_plan_rejects_bad_arguments(gk):
    mesh = gk.generate_sphere_mesh(1.0, 1)
    with pytest.raises(gk.InvalidArgument):
        gk.edge_blocks_plan(mesh, 0)
    with pytest.raises(gk.InvalidArgument):
        gk.edge_blocks_plan(mesh, 13)
    with pytest.raises(gk.InvalidArgument):
        gk.edge_blocks_plan(mesh, 4, 2)
