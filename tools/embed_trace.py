"""Phases of one embed() call on a BASELINE configuration (GEMPE_TRACE=1 prints the laps of construction, run and export):

    GEMPE_TRACE=1 python tools/embed_trace.py [c4]
"""
import os, sys, time, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_03479_b200 as P
from paper_2011_03479_b200 import graphgen
n, src, dst, dim, k, _, init, std = graphgen.make_config(sys.argv[1] if len(sys.argv) > 1 else 'c4', device=torch.device('cuda', 0))
s, d = np.ascontiguousarray(src, np.uint32), np.ascontiguousarray(dst, np.uint32)
cfg = P.IterationConfig(max_iters=20, convergence_window=21)
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    t0 = time.perf_counter()
    g = P.Graph(n, s, d)
    t1 = time.perf_counter()
    e = P.EmbeddingEngine(g, dim, cfg, 1)
    t2 = time.perf_counter()
    r = e.run()
    t3 = time.perf_counter()
    e.close()
    print(f'graph {t1-t0:.3f} engine {t2-t1:.3f} run {t3-t2:.3f} total {t3-t0:.3f}', flush=True)
