"""Debug K = 4 chains: one small heat3d run with the chain forced on (run under
compute-sanitizer on a GPU box)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses

from oracle.oracle import bits_equal, strict_execute_dag
from paper_2512_19851_b200 import temporal
from paper_2512_19851_b200.programs import DagProgram, heat3d_program
from paper_2512_19851_b200.session import run_program

temporal.VALIDATED_K = (2, 4)
temporal.MIN_POINTS = 0
temporal.ENABLED = True
n, iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40, 8
temporal.DEFAULT = dataclasses.replace(temporal.DEFAULT, k=4, bx=32, by=32)
prog = DagProgram()
heat3d_program(prog, n, iters, seed_fills=6)
want = strict_execute_dag(prog.dag, prog.shapes)
job, _ = run_program(prog)
ok = all(bits_equal(job.fetch(a), want[a]) for a in prog.shapes)
print("K=4 ran:", bool(job.executors[0]._scratch), "bit-exact:", ok)
job.close()
