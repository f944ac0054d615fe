import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from helpers import gaussian_qkv, to_dev, rel_l2, bf16_round
from oracle import psa_oracle as orc
import paper_2512_04025_b200 as psa
n, d, b, H = 1024, 128, 128, 4
q, k, v = gaussian_qkv(11, 1, n, d)
nb = n // b
lay = psa.make_layout(n, d, b, b, H); olay = orc.Layout(n, d, b, b, H)
pyr = psa.build_pyramid(to_dev(k), to_dev(v), lay)
kl, vl = orc.build_pyramid(k[0], v[0], olay)
for name, m in [("all1", np.ones((nb, nb), int)), ("all2", np.full((nb, nb), 2)), ("all3", np.full((nb, nb), 3)),
                ("all4", np.full((nb, nb), 4)), ("one1", np.eye(nb, dtype=int)), ("one2", 2 * np.eye(nb, dtype=int)),
                ("mix12", np.tile([1, 2], (nb, nb // 2)))]:
    res = psa.psa_streaming(to_dev(q[0]), pyr, torch.from_numpy(m).cuda())
    out = res.out.float().cpu().numpy().astype(np.float64)
    lse = res.row_log_normalizers.cpu().numpy()
    ro, rl, sk = orc.psa_materialized(q[0], [bf16_round(x) for x in kl], [bf16_round(x) for x in vl], m, olay)
    print(name, 'rel', rel_l2(out, ro), 'lse err mean', (lse - rl).mean(), 'max', np.abs(lse - rl).max())
