"""Two stream-K launches on two streams at once. Their tail owners spin on
flags other clusters publish, so each launch needs all of its CTAs resident;
launched cooperatively, the second waits for SMs instead of splitting them
with the first (which could leave both waiting on CTAs that cannot be
scheduled). Runs in a subprocess with a timeout so a regression fails the
test instead of hanging the session. Integer inputs: both results exact."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import sys; sys.path.insert(0, {root!r})
import numpy as np, torch
import paper_2003_06324_b200 as fi

def setup(m, n, k, **kw):
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, pair=True, tile_n=256, **kw))
    g = torch.Generator(device="cuda").manual_seed(m + k)
    A = torch.randint(-3, 4, (k, m), device="cuda", generator=g).half()
    B = torch.randint(-3, 4, (n, k), device="cuda", generator=g).half()
    C = torch.empty(n * m, device="cuda")
    return plan, A, B, C, m, n

jobs = [setup(4096, 4096, 4096), setup(1024, 1024, 32768, split_k=4)]
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
for (plan, A, B, C, m, n) in jobs:  # workspaces allocated
    plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), 0)
torch.cuda.synchronize()
for rep in range(10):
    for (plan, A, B, C, m, n), s in zip(jobs, streams):
        plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
ok = True
rng = np.random.default_rng(0)
for (plan, A, B, C, m, n) in jobs:
    rows, cols = rng.integers(0, m, 256), rng.integers(0, n, 256)
    ri, ci = torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda()
    a = A[:, ri].T.double(); b = B[ci, :].double()
    want = (a * b).sum(1)
    got = C.view(n, m)[ci, ri].double()
    ok = ok and bool(torch.equal(got, want))
print("OK" if ok else "MISMATCH")
"""


def test_two_stream_k_launches_on_two_streams():
    r = subprocess.run([sys.executable, "-c", CODE.format(root=ROOT)], capture_output=True, text=True, timeout=120)
    assert r.stdout.strip().endswith("OK"), r.stdout + r.stderr
