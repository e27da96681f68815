"""C ABI: the in-tree library loads and exports every entry point the header
declares; host-only entry points (trees, point generators, seeds, shard plan)
agree with the CPU oracle.  No device is touched here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bfly_b200.h")
LIB = os.path.join(ROOT, "paper_2002_03400_b200", "_native", "libbfly_b200.so")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(bfly_[a-z0-9_]+)\s*\(", src))
    names.discard("bfly_apply_fn")
    return sorted(names)


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "run __graft_entry__.build() first"
    lib = C.CDLL(LIB)
    names = declared_functions()
    assert len(names) > 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_seed_mix_and_points_match_oracle():
    import paper_2002_03400_b200 as B

    for seed, words in ((0, ()), (0, (1, 2)), (12345, (3, 7, 1)), (2**63 + 5, (6, 1, 0, 9))):
        assert B.seed_mix(seed, *words) == O.seed_mix(seed, *words)
    for n in (1, 7, 1000):
        a = B.configs.points_uniform(n, 3, 2, -n / 2, n / 2)
        b = np.zeros((n, 3))
        O.lib().bo_points_uniform(n, 3, 2, -n / 2, n / 2, O._ptr(b))
        assert np.array_equal(a, b)
        a = B.configs.points_half_circle(n, False)
        O.lib().bo_points_half_circle(n, 0, O._ptr(b))
        assert np.array_equal(a, b)
    a = B.configs.points_plate(16, 2.0)
    b = np.zeros((256, 3))
    O.lib().bo_points_plate(16, 2.0, O._ptr(b))
    assert np.array_equal(a, b)


@pytest.mark.parametrize("dim,n,L", [(1, 37, 3), (2, 64, 4), (3, 1000, 5), (2, 4096, 7)])
def test_tree_matches_oracle(dim, n, L):
    """tree.hpp:75-201 (longest axis, stable sort, left child ceil)."""
    import paper_2002_03400_b200 as B

    rng = np.random.default_rng(n)
    pts = np.zeros((n, 3))
    pts[:, :dim] = rng.random((n, dim))
    pts[::7, 0] = 0.5  # ties: stability matters
    t = B.PartitionTree.build(pts[:, :dim], L)
    o = O.PartitionTree.build(pts[:, :dim], L)
    assert np.array_equal(t.perm, o.perm)
    assert np.array_equal(t.flat_ranges, o.range_flat)
    # test_tree.cpp:86-98: rebuilding on tree-ordered points is the identity
    t2 = B.PartitionTree.build(pts[t.perm][:, :dim], L)
    assert np.array_equal(t2.perm, np.arange(n))


def test_tree_errors_and_depth():
    import paper_2002_03400_b200 as B

    with pytest.raises(B.PreconditionError):
        B.PartitionTree.build(np.arange(8.0), 4)  # 2^L > n (test_tree.cpp:26)
    with pytest.raises(B.PreconditionError):
        B.PartitionTree.build(np.array([0.0, np.nan, 1.0, 2.0]), 1)
    for n, leaf in ((4096, 32), (65536, 32), (262144, 64), (16384, 32), (100, 3)):
        assert B.PartitionTree.depth_for(n, leaf) == O.depth_for(n, leaf)
    t = B.PartitionTree.build(np.arange(8.0), 1)
    assert t.node_range(1, 0) == (0, 4) and t.node_range(1, 1) == (4, 8)


def test_config_defaults_match_reference():
    """ReconstructionConfig defaults (reconstruct.hpp:10-20)."""
    import paper_2002_03400_b200 as B

    c = B.ReconstructionConfig()
    assert (c.tolerance, c.oversampling, c.rank_guess, c.center, c.hard_cap, c.threads) == (1e-6, 2, 4, -1, -1, 1)
    assert B.ReconstructionConfig(levels=7).center_level() == 3
