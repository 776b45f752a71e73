"""Region graphs and the layered plan (reference tests/test_structures.py and
tests/test_compiler.py re-targeted at this package)."""

import itertools
import json

import pytest

from paper_2004_06231_b200.compiler import (EinsumLayer, LeafLayer, MixingLayer, assign_replica,
                                            compile_graph, topological_layers)
from paper_2004_06231_b200.structures import (Partition, Region, RegionGraph, Scope,
                                              StructureConfig, lift_channels, poon_domingos,
                                              random_binary_tree, validate)


def test_binary_tree_minimal():
    rg = random_binary_tree(2, StructureConfig(depth=1, replicas=1, seed=0))
    assert len(rg.partitions) == 1
    assert {rg.regions[r].scope for r in rg.leaf_region_ids()} == {Scope([0]), Scope([1])}


def test_binary_tree_replicas_and_validity():
    rg = random_binary_tree(512, StructureConfig(depth=4, replicas=10, seed=3))
    assert len(rg.child_partitions(rg.root)) == 10
    assert len(rg.leaf_region_ids()) == 10 * 2 ** 4
    assert validate(rg) == []


def test_binary_tree_rejects_overdeep():
    with pytest.raises(ValueError):
        random_binary_tree(4, StructureConfig(depth=3, replicas=1, seed=0))


def test_binary_tree_path_depth():
    rg = random_binary_tree(16, StructureConfig(depth=3, replicas=2, seed=5))
    parent = {c: p.parent for p in rg.partitions.values() for c in (p.left, p.right)}
    for leaf in rg.leaf_region_ids():
        steps, node = 0, leaf
        while node != rg.root:
            node, steps = parent[node], steps + 1
        assert steps == 3


def test_pd_enumeration_and_contiguity():
    rg = poon_domingos(2, 2, StructureConfig(deltas=(1,), axes="both"))
    assert len(rg.regions) == sum((3 - h) * (3 - w) for h, w in itertools.product((1, 2), (1, 2)))
    rg = poon_domingos(3, 4, StructureConfig(deltas=(1, 2), axes="both"))
    assert validate(rg) == []
    for r in rg.regions.values():
        rows = sorted({v // 4 for v in r.scope})
        cols = sorted({v % 4 for v in r.scope})
        assert len(r.scope) == len(rows) * len(cols)


def test_lift_channels_keeps_validity():
    rg = lift_channels(poon_domingos(4, 4, StructureConfig(deltas=(2,), axes="both")), 3)
    assert rg.d_vars == 48 and validate(rg) == []
    assert all(len(r.scope) % 3 == 0 for r in rg.regions.values())


def test_validate_violations():
    rg = RegionGraph(d_vars=3)
    rg.regions[0] = Region(0, Scope([0, 1, 2]))
    rg.regions[1] = Region(1, Scope([0, 1]))
    rg.regions[2] = Region(2, Scope([1, 2]))
    rg.partitions[3] = Partition(3, 0, 1, 2)
    assert any("decomposability" in v for v in validate(rg))
    rg.regions[2] = Region(2, Scope([1]))
    assert any("completeness" in v for v in validate(rg))
    rg.regions[9] = Region(9, Scope([2]))
    assert any("unreachable" in v for v in validate(rg))


def test_json_round_trip():
    rg = poon_domingos(2, 3, StructureConfig(deltas=(1,), axes="both"))
    assert RegionGraph.from_json(rg.to_json()).to_json() == rg.to_json()


def test_layering_and_cycle():
    rg = random_binary_tree(4, StructureConfig(depth=2, replicas=2, seed=1))
    layers = topological_layers(rg)
    pos = {n: i for i, layer in enumerate(layers) for n in layer}
    for p in rg.partitions.values():
        assert pos[p.left] < pos[p.id] < pos[p.parent]
    bad = RegionGraph(d_vars=2)
    bad.regions[0] = Region(0, Scope([0, 1]))
    bad.regions[1] = Region(1, Scope([0]))
    bad.regions[2] = Region(2, Scope([1]))
    bad.partitions[3] = Partition(3, 0, 1, 2)
    bad.partitions[4] = Partition(4, 1, 0, 2)
    with pytest.raises(ValueError):
        topological_layers(bad)


def test_replica_assignment():
    assert assign_replica(poon_domingos(1, 4, StructureConfig(deltas=(2,), axes="vertical"))).count == 1
    assert assign_replica(random_binary_tree(16, StructureConfig(depth=2, replicas=10, seed=2))).count == 10


def test_compile_plan_properties():
    rg = random_binary_tree(8, StructureConfig(depth=1, replicas=3, seed=0))
    c = compile_graph(rg, k=2)
    mixes = [l for l in c.layers if isinstance(l, MixingLayer)]
    assert len(mixes) == 1 and mixes[0].is_root and mixes[0].mask.sum() == 3
    rg = random_binary_tree(8, StructureConfig(depth=2, replicas=2, seed=4))
    c = compile_graph(rg, k=3, k_root=1)
    for layer in c.layers[1:]:
        assert all(r == -1 or 0 <= r < c.num_buffer_rows for r in layer.out_rows)
    assert c.layers[-1].is_root
    rg = poon_domingos(2, 3, StructureConfig(deltas=(1,), axes="both"))
    owners = [o for l in compile_graph(rg, 2).layers if isinstance(l, EinsumLayer) for o in l.owners]
    assert sorted(pid for _, pid in owners) == sorted(rg.partitions)
    doc = json.loads(compile_graph(rg, 2).plan_json())
    assert doc["layers"][0]["type"] == "leaf"
    with pytest.raises(ValueError):
        compile_graph(rg, k=0)
    lone = RegionGraph(d_vars=1)
    lone.regions[0] = Region(0, Scope([0]))
    with pytest.raises(ValueError):
        compile_graph(lone, k=2)
