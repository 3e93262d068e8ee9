"""The library's own launch count (imq_ext_stats.kernel_launches, reported by
bench.py as gpu_launches) against the kernels a profiler sees in one product."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("t, L", [(0.01, 5), (0.2, 5), (0.05, 6)])
def test_kernel_launch_count_matches_profiler(imq, t, L):
    torch = pytest.importorskip("torch")
    from torch.profiler import ProfilerActivity, profile
    from paper_2205_04194_b200 import inputs
    n = 1 << 18
    xy = inputs.uniform_points(n, 0)
    u = torch.tensor(inputs.random_vector(n, 3), device="cuda")
    b = torch.empty_like(u)
    with imq.FastOperator(xy, t, 12, L) as op:
        op.apply_device(u, b)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            op.apply_device(u, b)
            torch.cuda.synchronize()
        st = op.stats()
    kernels = [e for e in prof.events() if e.device_type.name == "CUDA"
               and "memset" not in e.name.lower() and "memcpy" not in e.name.lower()]
    # every kernel of a product is this library's own (no cuBLAS / CUB / torch)
    assert all("imqk" in e.name for e in kernels), sorted({e.name[:60] for e in kernels})
    assert len(kernels) == st["kernel_launches"], (len(kernels), st,
                                                   sorted({e.name[:60] for e in kernels}))
