"""Pair split-K over a 4-CTA cluster (DSMEM reduction, instance (2,256,2)): exact on integers?"""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import numpy as np
import paper_2003_06324_b200 as fi
import oracle
m, n, k = 4096, 4096, 512
plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, split_k=2))
print("cluster", plan.info.cluster, "splitk_global?", plan.info.streamk)
a = oracle.fill(m, k, 3, True); b = oracle.fill(k, n, 4, True)
c = plan.run_host(a, b)
rng = np.random.default_rng(0); rows, cols = rng.integers(0, m, 2000), rng.integers(0, n, 2000)
want = oracle.sample_f64(oracle.round_elem(a, "f16"), oracle.round_elem(b, "f16"), rows, cols)
got = c[rows, cols]
print("exact fraction", np.mean(got == want))
# by CTA pair: rows within 256-row tile [0,128) vs [128,256) and split rank? print error by row block
bad = got != want
print("bad rows mod 256 < 128:", np.mean(bad[rows % 256 < 128]), ">=128:", np.mean(bad[rows % 256 >= 128]))
