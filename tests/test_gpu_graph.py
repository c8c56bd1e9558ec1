"""Plans captured in a CUDA graph and replayed with new inputs. The K-slice
tail fixups synchronise through epoch flags; a host-side epoch would be frozen
at capture, so every replay after the first would take the previous replay's
partials as published. The epoch therefore lives on the device (advanced by the
last CTA of each launch). Integer inputs: every replay exact."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [  # m, n, k, strategy kwargs: the pull fixup (C2), symmetric + remainder (C3), N-split
    (4096, 4096, 4096, dict()),
    (1024, 1024, 32768, dict(split_k=4)),
    (2560, 2560, 8192, dict()),
]


def _check(torch, A, B, C, m, n, seed):
    rng = np.random.default_rng(seed)
    rows, cols = rng.integers(0, m, 512), rng.integers(0, n, 512)
    ri, ci = torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda()
    a = A[:, ri].T.float().cpu().numpy().astype(np.float64)
    b = B[ci, :].float().cpu().numpy().astype(np.float64)
    want = np.einsum("sk,sk->s", a, b)
    got = C.view(n, m)[ci, ri].cpu().numpy().astype(np.float64)
    return np.array_equal(got, want)


@pytest.mark.parametrize("m,n,k,kw", CASES)
def test_graph_replay_with_new_inputs(fi, m, n, k, kw):
    import torch
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, pair=True, tile_n=256, **kw))
    A = torch.zeros((k, m), device="cuda", dtype=torch.float16)   # col-major M x K
    B = torch.zeros((n, k), device="cuda", dtype=torch.float16)   # col-major K x N
    C = torch.empty(n * m, device="cuda")
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):  # warm-up outside the capture (workspace allocation)
        plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), side.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), torch.cuda.current_stream().cuda_stream)
    gen = torch.Generator(device="cuda")
    for trial in range(4):
        gen.manual_seed(100 + trial)
        A.copy_(torch.randint(-3, 4, A.shape, device="cuda", generator=gen).half())
        B.copy_(torch.randint(-3, 4, B.shape, device="cuda", generator=gen).half())
        g.replay()
        torch.cuda.synchronize()
        assert _check(torch, A, B, C, m, n, trial), f"replay {trial}"


def test_first_launch_inside_a_capture_is_refused(fi):
    """The stream-K workspace cannot be allocated inside a capture (it would be
    graph-owned memory): the launch fails with a clear error instead."""
    import torch
    plan = fi.Plan(fi.strategies.tc_strategy(4096, 4096, 4096))  # pull-fixup tail: needs a workspace
    A = torch.zeros((4096, 4096), device="cuda", dtype=torch.float16)
    C = torch.empty(4096 * 4096, device="cuda")
    g = torch.cuda.CUDAGraph()
    with pytest.raises(fi.FiError) as e:
        with torch.cuda.graph(g):
            plan.launch(A.data_ptr(), A.data_ptr(), C.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert "outside" in str(e.value)
