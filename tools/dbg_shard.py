import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2209_04626_b200 as mp, oracle, testmat
a = testmat.config_matrix("C3", 333)
uo, so, vo, sto, rc = oracle.mixed_svd(a, b=32)
d = np.linalg.norm(a, axis=0); s = np.linalg.svd(a / d, compute_uv=False); k = s[0] / s[-1]
def dev(x): return torch.from_numpy(np.asfortranarray(x)).cuda().t().contiguous().t()
for opts in [dict(), dict(qrp_panel_stages=0), dict(gram_pdl=0), dict(qrp_panel_stages=0, gram_pdl=0)]:
    for G in (1, 2):
        U, S, V, st = mp.factor(dev(a), block_cols=32, virtual_shards=G, **opts)
        S = S.cpu().numpy(); U = U.cpu().numpy(); V = V.cpu().numpy()
        rel = np.abs(S - so) / so
        u64 = 2.0 ** -53
        ratio = np.max(np.abs(S - so) / (u64 * np.minimum(k, so[0] / so) * so))
        print(opts, G, "rc", st["rc"], "sw", st["sweeps32"], st["sweeps64"], "oracle", sto["sweeps32"], sto["sweeps64"],
              "maxrel %.2e ratio %.1f" % (rel.max(), ratio), "orthU %.1e" % np.abs(U.T @ U - np.eye(333)).max(),
              "res %.1e" % (np.linalg.norm(a - (U * S) @ V.T) / np.linalg.norm(a)))
