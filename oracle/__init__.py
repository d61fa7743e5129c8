"""ED-Batch CPU oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU implementations of what the hot path computes, written
from PAPER.md (arXiv 2302.03851) and the readings listed in DESIGN.md §3:

  oracle.graph     merged DAG, frontier, typed subgraphs, depth, lower bound (App. B.3)
  oracle.schedule  Alg. 1 FSM batching with E_sort/E_base/E_max, depth/agenda/SC heuristics,
                   brute-force optimum, FSM-table enumeration
  oracle.layout    schedule-order layout, PQ/C1P layout planner, check_ideal (App. C)
  oracle.cells     fp64 cell equations (SURVEY App. A readings; the paper only cites them)
  oracle.evaluate  fp64 per-node recursive evaluator + level-synchronous evaluator

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
import anything here.  The product path (paper_2302_03851_b200/) never imports this package
and shares no code with it: the only shared module is workloads/ (seeded input generators,
none of the method's arithmetic).
"""
