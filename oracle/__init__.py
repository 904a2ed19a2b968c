"""fp64 CPU oracle of the expert-parallel MoE layer (arxiv 2605.05049, "Piper").

TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``.  The product
package ``paper_2605_05049_b200`` never imports it, and the two share no code:
no kernels, headers, helpers, tables or constant generators.  Inputs come from
``synth`` (seeded generators only, none of the method's arithmetic).

Modules
  moe_ref   the layer, step by step in the paper's notation (Table II)
  counters  FLOP / byte counters evaluated from the realised routing
  migration Alg. 2 expert migration (NEXT-2)
  dedup     per-destination-rank deduplicated all-to-all (NEXT-4, reading R18)
  pipeline  1F1B schedule of the PP x EP executor and Eq. 4's activation term (NEXT-3, R19)

Parity pins: see tests/test_oracle_*.py; "parity unpinned" items are listed in
DESIGN.md §Oracle and in the docstrings below.
"""
from . import moe_ref, counters, dedup, pipeline  # noqa: F401
