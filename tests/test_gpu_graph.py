"""fft_exec inside a CUDA graph (an exec is launches only —
the pipelined kernel's counters reset themselves, its tensor map is encoded at
capture time): capture once, replay with new input contents, compare with
direct execs (bit-identical) and with the oracle."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

bf = pytest.importorskip("paper_1407_6915_b200")


@pytest.mark.parametrize("n,b", [(1024, 64), (1 << 13, 449), (1 << 14, 300), (1 << 16, 37), (1 << 20, 5)])
def test_exec_replayed_from_a_cuda_graph(n, b):
    x = torch.empty((b, n), dtype=torch.complex64, device="cuda")
    y = torch.empty_like(x)
    with bf.Plan(n, b) as p:
        x.copy_(torch.from_numpy(synth.random_records(5, n, 0, b)))
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            p.exec(x, y)                    # warm-up outside capture
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            p.exec(x, y)
        for seed in (11, 12, 13):
            h = synth.random_records(seed, n, 0, b)
            x.copy_(torch.from_numpy(h))
            g.replay()
            torch.cuda.synchronize()
            got = y.cpu().numpy()
            y_direct = torch.empty_like(x)
            p.exec(x, y_direct)
            torch.cuda.synchronize()
            assert np.array_equal(got, y_direct.cpu().numpy()), seed
            rows = [0, b // 2, b - 1]
            err = oracle.rel_l2(got[rows], oracle.records_c64(h[rows], oracle.FORWARD))
            assert np.all(err <= oracle.tolerance(n)), (seed, err.max())
