"""Collected with the reference suite (tests/test_gpu_reference_suite.py): proves the
shim routes the reference's imports to this package and its CUDA library."""


def test_kvfuse_hot_path_is_the_device_package():
    import kvfuse
    import kvfuse.attention
    import kvfuse.core
    import kvfuse.fusion
    from paper_2601_03067_b200 import _native

    assert kvfuse.__shim__
    assert kvfuse.fusion.fuse_batch.__module__ == "paper_2601_03067_b200.fusion"
    assert kvfuse.core.PagedKvCache.__module__ == "paper_2601_03067_b200.core"
    assert kvfuse.attention.paged_attention.__module__ == "paper_2601_03067_b200.attention"
    assert kvfuse.fuse_chunks.__module__ == "paper_2601_03067_b200.fusion"
    assert _native.lib() is not None and _native.LIB_PATH.exists()
    from kvfuse.workload import generate_fixture

    cache = generate_fixture("clusters4")
    assert type(cache).__module__ == "paper_2601_03067_b200.core"
    assert cache.keys_dev is not None and cache.keys_dev.is_cuda
