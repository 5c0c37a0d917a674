"""GPU parity of the one-process multi-GPU entry (qg_host_mul_common_multi,
paper_0803_1975_b200/csrc/qg_multi.cpp): row shards over the process's
devices, B packed once and broadcast as packed words by ncclBroadcast, C
gathered to the host — against the oracle's naive_gemm (gemm.hpp:80-100).
On a one-GPU box the device list repeats nothing: it is [0] (a one-rank NCCL
communicator, the same code path as N ranks)."""
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
