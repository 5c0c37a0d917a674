"""GPU parity of the one-process multi-GPU entry (qg_host_mul_common_multi,
paper_0803_1975_b200/csrc/qg_multi.cpp): row shards over the process's
devices, every device packing only its tile-column slot of B and one grouped
in-place ncclAllGather assembling the packed CB_t, C gathered to the host —
against the oracle's naive_gemm (gemm.hpp:80-100). On a one-GPU box the
device list is [0] (a one-rank NCCL communicator, the same code path as N
ranks). Also the multi-process host entry (dist.mul_common_allgather_host)
at world size 1 and the host API across two devices of one thread."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p,m,k,n", [(7, 1000, 4096, 515), (3, 70, 300, 50), (5, 129, 2000, 4099), (3, 1, 7, 1)])
def test_multi_matches_oracle(qg, orc, cuda, p, m, k, n):
    import torch

    devices = list(range(torch.cuda.device_count()))
    a = orc.random_residue_matrix(m, k, p, 31)
    b = orc.random_residue_matrix(k, n, p, 32)
    want = orc.naive_gemm(p, a, b)
    for plan in (qg.plan_gpu(p, k), qg.plan_gpu(p, k, balanced=False)):
        assert np.array_equal(qg.mul_common_multi_host(a, b, plan, devices), want)


def test_multi_config2_checksum(qg, orc, cuda):
    """BASELINE config 2 through the multi-GPU entry: the reference's checksum."""
    import torch

    p, m, k, n = 7, 4096, 4096, 4096
    a = qg.random_residue_matrix(m, k, p, 42, dtype=torch.int32).cpu().numpy().view(np.uint32)
    b = qg.random_residue_matrix(k, n, p, 43, dtype=torch.int32).cpu().numpy().view(np.uint32)
    c = qg.mul_common_multi_host(a, b, qg.plan_gpu(p, k), list(range(torch.cuda.device_count())))
    assert qg.residue_checksum(c) == 50333685


def test_multi_errors(qg, cuda):
    a = np.zeros((4, 4), np.uint32)
    with pytest.raises(qg.InvalidArgument):
        qg.mul_common_multi_host(a, a, qg.plan_gpu(3, 4), [])


@pytest.mark.parametrize("p,m,k,n", [(7, 1000, 4096, 515), (3, 300, 32768, 256), (5, 129, 2000, 4099)])
def test_allgather_host_entry_world1(qg, orc, cuda, p, m, k, n):
    """dist.mul_common_allgather_host (B slot packed from host, gathered CB_t,
    A streamed against it) at world size 1 equals naive_gemm."""
    from paper_0803_1975_b200.dist import mul_common_allgather_host

    a = orc.random_residue_matrix(m, k, p, 3)
    b = orc.random_residue_matrix(k, n, p, 4)
    assert np.array_equal(mul_common_allgather_host(a, b, qg.plan_gpu(p, k), 0, 1), orc.naive_gemm(p, a, b))


def test_host_api_on_two_devices_one_thread(qg, orc, cuda):
    """The pipelined host API keeps one stream set per device: the
    same thread calls it on device 0, then on device 1, then on 0 again."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    p, m, k, n = 7, 600, 4096, 300
    a = orc.random_residue_matrix(m, k, p, 5)
    b = orc.random_residue_matrix(k, n, p, 6)
    want = orc.naive_gemm(p, a, b)
    for dev in (0, 1, 0):
        torch.cuda.set_device(dev)
        assert np.array_equal(qg.mul_common_compressed_host(a, b, qg.plan_gpu(p, k)), want), dev
    torch.cuda.set_device(0)
