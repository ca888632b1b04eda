"""Fixture -> product-object helpers shared by the test modules."""

from __future__ import annotations

import numpy as np

from conftest import graph_keys, jload, labels_from, load, params_from


def product_graph(fx, prefix="g_"):
    from paper_2109_07893_b200 import DynamicGraph, SparseMatrix
    n, snaps = graph_keys(fx, prefix)
    return DynamicGraph(n, [SparseMatrix.from_canonical(n, r, c, v) for r, c, v in snaps])


def product_case(name):
    """(fx, cfg, data, train LabelSet, test LabelSet, params) for a model fixture."""
    import paper_2109_07893_b200 as pk
    fx = load(name)
    meta = jload(fx["cfg"])
    cfg = pk.ModelConfig(architecture=meta["architecture"], in_features=2, hidden_features=meta["hidden"],
                         embed_features=meta["hidden"], window=meta["window"])
    g = product_graph(fx)
    data = pk.prepare_training_data(cfg, g)
    train = pk.LabelSet(2, labels_from(fx, "train_"))
    test = pk.LabelSet(2, labels_from(fx, "test_"))
    params = params_from(fx, "p_")
    return fx, cfg, data, train, test, params
