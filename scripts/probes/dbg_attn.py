import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from helpers import gaussian_qkv, to_dev, rel_l2, bf16_round
from oracle import psa_oracle as orc
import paper_2512_04025_b200 as psa
for (n, d, b, H) in [(1024, 64, 64, 4), (1920, 128, 120, 4), (1024, 128, 128, 4)]:
    rng = np.random.default_rng(20240911)
    q, k, v = gaussian_qkv(11, 2, n, d)
    nb = n // b
    mask = rng.integers(0, H + 1, size=(2, nb, nb))
    mask[0, 0, :] = 0
    mask[1, 1, :] = 0
    mask[1, 1, 2] = 1
    lay = psa.make_layout(n, d, b, b, H); olay = orc.Layout(n, d, b, b, H)
    pyr = psa.build_pyramid(to_dev(k), to_dev(v), lay)
    res = psa.psa_streaming(to_dev(q), pyr, torch.from_numpy(mask).cuda())
    out = res.out.float().cpu().numpy().astype(np.float64)
    lse = res.row_log_normalizers.cpu().numpy()
    for h in range(2):
        kl, vl = orc.build_pyramid(k[h], v[h], olay)
        ro, rl, sk = orc.psa_materialized(q[h], [bf16_round(x) for x in kl], [bf16_round(x) for x in vl], mask[h], olay)
        err = np.abs(out[h] - ro)
        r = np.unravel_index(err.argmax(), err.shape)
        rowerr = err.max(axis=1)
        bad = np.nonzero(rowerr > 1e-2 * np.abs(ro).max())[0]
        fin = np.isfinite(rl)
        print((n,d,b,H), h, 'rel', rel_l2(out[h], ro), 'maxabs', err.max(), 'at', r, 'ref max', np.abs(ro).max(),
              'bad rows', bad[:20], len(bad), 'lse err', np.abs(lse[h][fin]-rl[fin]).max())
        if len(bad):
            i = bad[0] // b
            print('  q-block', i, 'mask row', mask[h, i].tolist())
            print('  got', out[h, bad[0], :6], 'ref', ro[bad[0], :6], 'lse', lse[h, bad[0]], rl[bad[0]])
