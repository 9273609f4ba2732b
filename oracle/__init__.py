"""fp64 CPU oracle for the ORBIT-2 TILES Reslim forward (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference legs) may import this package.  See reslim_tiles.py.
"""
from .reslim_tiles import *  # noqa: F401,F403
from .reslim_tiles import Problem, Tile, plan_tiles, tiles_forward, tiles_forward_sampled, global_forward  # noqa: F401
