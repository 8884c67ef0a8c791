"""Multi-round pin of the CUDA path: R rounds of Alg. 1 through smcsd_step (S1-S7 + bonus
token) and smcsd_kv_reindex (S9, the in-place slot plan applied to the token histories on the
device) satisfy SMC's unbiasedness identity E[Z_R sum_n wbar_n phi(x_n)] = E_p[phi] on a toy
Markov LM with exact p (tests/smc_rounds.py) -- the same pin the oracle passes in
test_oracle_rounds.py, checked independently of it."""
import math

import numpy as np
import pytest
import torch

import smc_rounds as sr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N,K,R,scheme", [(8, 1, 2, 0), (4, 2, 2, 0), (16, 1, 3, 0), (8, 1, 2, 1)])
def test_gpu_multi_round_unbiased(N, K, R, scheme):
    import paper_2604_15672_b200 as smc
    dev = torch.device("cuda")
    P = 6000
    p_tab, q_tab = sr.tables()
    ws = smc.Workspace(dev)

    def backend(r, lp, lq, tok, eta):
        prev = torch.full((P, N), float(-math.log(N)), dtype=torch.float32, device=dev)
        out = smc.smcsd_step(torch.from_numpy(lp).to(dev), torch.from_numpy(lq).to(dev),
                             torch.from_numpy(tok).to(dev), V=sr.V, logw_prev=prev, eta=eta,
                             scheme=scheme, seed=0x5EED5EED, step=r, bonus=True, workspace=ws)
        torch.cuda.synchronize()
        assert int(out.status.abs().sum()) == 0
        return (out.lse.cpu().numpy(), out.bonus.cpu().numpy(), out.slot_src.cpu().numpy(),
                out.logw_pre.cpu().numpy())

    def reindex(hist, slot_src):
        T = hist.shape[2]
        Tp = (T + 3) // 4 * 4                                   # rows padded to 16-byte multiples
        h = torch.zeros((P, N, Tp), dtype=torch.int32, device=dev)
        h[:, :, :T] = torch.from_numpy(np.ascontiguousarray(hist)).to(dev)
        smc.smcsd_kv_reindex(h, h, torch.from_numpy(slot_src).to(dev), n_outer=1, outer_stride=0,
                             prompt_stride=N * Tp * 4, particle_stride=Tp * 4, seg_count=1,
                             seg_bytes=Tp * 4, seg_stride=Tp * 4)
        return h[:, :, :T].cpu().numpy()
    log_z, hist, wbar = sr.run(backend, reindex, P=P, N=N, K=K, R=R, seed=11, p_tab=p_tab, q_tab=q_tab)
    ev, ps = sr.exact_events(p_tab, R * (K + 1))
    est, se = sr.estimate(log_z, hist, wbar, ev)
    z = (est - ps) / se
    assert np.max(np.abs(z)) < 5.0, (np.max(np.abs(z)), ev[int(np.argmax(np.abs(z)))])
    assert float(np.sum(z ** 2)) < 3.0 * len(ev)
