"""TEST INFRASTRUCTURE ONLY -- the float64 CPU oracle for GSASR rasterization.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package. The product path
(paper_2501_06838_b200) never imports it and shares no code with it.
"""
from .oracle import (OracleLib, build_oracle, out_dims, render_fwd, render_bwd, render_pixels,
                     field, rects, pair_count, tile_lists, load)

__all__ = ["OracleLib", "build_oracle", "out_dims", "render_fwd", "render_bwd", "render_pixels",
           "field", "rects", "pair_count", "tile_lists", "load"]
