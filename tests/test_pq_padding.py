"""General p/q implicit padding.

CPU: the oracle's implicit p/q transform (O3) against the explicitly padded
DFT of the same data (the definition), its round trip (qm U exactly), and
the p/q convolution against the D1 direct sums.  GPU: idc_cconv1d_pq."""
import numpy as np
import pytest

import synthgen
from oracle import dft_matrix, direct, implicit, rel_l2

PQ = [(1, 2), (1, 3), (2, 4), (2, 5), (3, 6), (3, 7), (3, 8)]


@pytest.mark.parametrize("p,q", PQ)
def test_pq_backward_is_the_padded_dft(p, q):
    m = 8
    U = synthgen.cconv1d_inputs(p * m, 2, roles=(0,))[0]
    S = implicit.fftpad_pq_backward(U, p, q)
    full = U @ dft_matrix(q * m, range(p * m), range(q * m), +1)     # u_j = sum_k zeta_qm^{jk} U_k
    for r in range(q):
        assert rel_l2(S[r], full[..., r::q]) < 1e-14
    back = implicit.fftpad_pq_forward(S, p, q, m)
    assert rel_l2(back, U) < 1e-14                                   # qm U / qm


@pytest.mark.parametrize("p,q", PQ)
def test_pq_convolution_is_d1(p, q):
    m = 8
    f, g = synthgen.cconv1d_inputs(p * m, 3)
    assert rel_l2(implicit.cconv1d_pq(f, g, p, q), direct.cconv1d(f, g)) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("p,q", PQ)
@pytest.mark.parametrize("m,B", [(8, 5), (64, 3), (1024, 2)])
def test_cconv1d_pq_gpu(p, q, m, B):
    import torch
    from paper_1008_1366_b200 import idconv
    f, g = synthgen.cconv1d_inputs(p * m, B)
    F, G = torch.from_numpy(f.copy()).cuda(), torch.from_numpy(g.copy()).cuda()
    idconv.cconv1d_pq(F, G, p, q)
    assert rel_l2(F.cpu().numpy(), direct.cconv1d(f, g)) < 1e-14


@pytest.mark.gpu
def test_pq_rejects_aliasing_choices():
    import torch
    from paper_1008_1366_b200 import idconv
    f = torch.zeros(3 * 8, dtype=torch.complex128, device="cuda")
    with pytest.raises(idconv.IdcError) as e:
        idconv.cconv1d_pq(f, f.clone(), 3, 5)                        # q < 2p would alias
    assert e.value.code == idconv.ERR_UNSUPPORTED
