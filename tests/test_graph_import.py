"""The CUDA-graph step helper imports on a CPU-only host (it binds to the
C-ABI library like ops.py; capture itself needs a GPU: test_gpu_graph.py)."""


def test_graph_module_imports():
    import paper_2412_09764_b200 as pkg
    g = pkg.graph
    assert hasattr(g, "MemoryLayerStepGraph")
    assert callable(g.MemoryLayerStepGraph.replay)
