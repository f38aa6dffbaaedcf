"""Drop-in mirror of the reference's `tmpsim` Python module.

`import paper_2305_16121_b200.tmpsim as t` exposes the same names as the
reference's `tmpsim._core` (proj/python/bindings.cpp:21-237): ModelSpec,
build_operator_sequence, build_block_graph, schedule_*, simulate, costs,
planner, ... implemented in C++ in liboases.so. On top of them the B200 build
adds measured execution (paper_2305_16121_b200.runtime).
"""
from ._core import *  # noqa: F401,F403
from ._core import __doc__  # noqa: F401
