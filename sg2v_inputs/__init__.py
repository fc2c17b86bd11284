"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the colour-coding method: it only builds
graphs (CSR arrays) and template edge lists.  Both sides (``oracle/`` and
``paper_2009_11665_b200/``) receive these arrays as plain inputs; neither side
imports the other.  Recipes follow SURVEY.md §8(d) and are restated in
DESIGN.md §"Input recipe".
"""
from .graphs import (  # noqa: F401
    CSR,
    csr_from_edges,
    erdos_renyi,
    rmat,
    rmat_1m_like,
    miami_like,
    orkut_like,
    graph500_like,
    BIG_GRAPHS,
    cycle_graph,
    path_graph,
    complete_graph,
    house_tail_graph,
    disjoint_union,
    degree_stats,
)
from .templates import (  # noqa: F401
    TEMPLATES,
    template_edges,
    path_template,
    star_template,
    random_tree,
    all_trees,
)
