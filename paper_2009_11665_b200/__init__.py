"""B200-native colour-coding hot path of SubGraph2Vec (arXiv:2009.11665).

The product is libsg2v.so (include/sg2v.h); this package is its thin Python
binding.  See DESIGN.md.
"""
from .sg2v import (  # noqa: F401
    F32, F64, U64, Graph, Options, Sg2vError, Template, Workspace, colorize, count, count_batch,
    workspace_bytes_batch, Comm, graph_load_partition, partition_rows,
    graph_load_csr, plan_describe, plan_describe_n, profile_enable, profile_read, template_build,
    workspace_bytes, version, lib, estimate, profile_read_launches, partition_relabel,
    graph_set_vertex_ids, profile_kernel_count,
)
