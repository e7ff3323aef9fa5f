"""NVLS allreduce backend: CUDA multicast object,
multimem.ld_reduce / multimem.st in the NVSwitch.  On this one-GPU box the
team has one device (rank 0 of 1): the create / add-device / bind / map
path, the multicast barrier and the multimem instructions all run, and the
result must equal the input (the sum over one rank).  With >= 2 GPUs,
test_gpu_multidevice-style runs cover the real reduction (bench.py N>1).
Skips when no multicast team can be formed (sccl_nvls_supported)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2008_08708_b200 import sccl  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def supported():
    if not sccl.nvls_supported(0, 1):
        pytest.skip("no multicast team can be formed on device 0 (on the one-GPU slice used here the "
                    "attribute is 1 but cuMulticastCreate returns CUDA_ERROR_INVALID_VALUE for every "
                    "configuration: tools/probes/multicast_probe.py)")


@pytest.mark.parametrize("dt,tdt", [(sccl.F32, torch.float32), (sccl.BF16, torch.bfloat16), (sccl.F16, torch.float16)])
def test_nvls_single_rank(supported, dt, tdt):
    n = 1 << 20
    x = torch.randn(n, device="cuda").to(tdt)
    nv = sccl.NvlsAllreduce(0, 1, n * x.element_size(), dt, device=0)
    out = torch.empty_like(x)
    for _ in range(3):  # back-to-back: the per-CTA arrival counters advance
        out.zero_()
        nv.launch(x, out)
        torch.cuda.synchronize()
        nv.check()
        assert torch.equal(out, x)
    ptr, nbytes = nv.buffer()
    assert nbytes == n * x.element_size() and ptr
    nv.close()


def test_nvls_rejects_bad_sizes(supported):
    with pytest.raises(sccl.InvalidArgumentError):
        sccl.NvlsAllreduce(0, 1, 1000, sccl.F32, device=0)
    with pytest.raises(sccl.InvalidArgumentError):
        sccl.NvlsAllreduce(0, 1, 4096, sccl.U8, device=0)
