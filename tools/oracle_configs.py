"""CPU oracle timings for the BASELINE configs on this machine's host cores:
T=1 (one process) and T=all (one process per dodecant / cube, up to the core count), wall clock,
one warm-up then best of 3 for the small configs; config 3 times single dodecants (11 s each) and
scales by the dodecant count (12 dodecants in parallel for T=all)."""
import json, os, sys, time
from concurrent.futures import ProcessPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
import oracle
from oracle import tables

ROWS = tables.DRT_HEMISPHERE


_CUBES = {}


def job(args):
    cfg, kind, b, k = args
    if cfg not in _CUBES:                      # once per process: the inputs are large to regenerate
        _CUBES[cfg] = synth.config_input(cfg)
    cube = _CUBES[cfg][b]
    if kind == "drt":
        oracle.drt_alg1(oracle.orient(cube, ROWS[k]))
    else:
        oracle.djt_alg3(oracle.orient(cube, tables.table(tables.TABLE_HEMISPHERE, "djt")[k]))
    return 0


def timed(jobs, workers, reps=3):
    best = 1e30
    for r in range(reps + 1):
        t0 = time.perf_counter()
        if workers == 1:
            for j in jobs:
                job(j)
        else:
            with ProcessPoolExecutor(workers) as ex:
                list(ex.map(job, jobs))
        dt = time.perf_counter() - t0
        if r > 0:
            best = min(best, dt)
    return best


cores = os.cpu_count() or 1
only = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]
specs = {c: v for c, v in {1: ("drt", 1, [0]), 2: ("drt", 1, range(12)), 4: ("djt", 1, [0]),
                           5: ("drt", 256, range(12))}.items() if c in only}
for cfg, (kind, nb, ks) in specs.items():
    jobs = [(cfg, kind, b, k) for b in range(nb) for k in ks]
    t1 = timed(jobs, 1, reps=1 if cfg == 5 else 3)
    ta = timed(jobs, min(cores, len(jobs)), reps=1 if cfg == 5 else 3)
    print(json.dumps({"config": cfg, "oracle_T1_ms": 1e3 * t1, "oracle_Tall_ms": 1e3 * ta, "cores": min(cores, len(jobs))}), flush=True)
if 3 not in only:
    sys.exit(0)
t1 = timed([(3, "drt", 0, 0)], 1, reps=1)
ta = timed([(3, "drt", 0, k) for k in range(12)], min(cores, 12), reps=1)
print(json.dumps({"config": 3, "oracle_T1_ms": 12e3 * t1, "oracle_T1_note": "12 x one dodecant",
                  "oracle_Tall_ms": 1e3 * ta * (12 / min(cores, 12)) if cores < 12 else 1e3 * ta,
                  "cores": min(cores, 12)}), flush=True)
