import sys, ctypes, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from helpers import gaussian_qkv, to_dev
import paper_2512_04025_b200 as psa
from paper_2512_04025_b200 import _lib
lib = _lib.load()
n, d, b, H = 1024, 128, 128, 4
q, k, v = gaussian_qkv(11, 1, n, d)
nb = n // b
lay = psa.make_layout(n, d, b, b, H)
pyr = psa.build_pyramid(to_dev(k), to_dev(v), lay)
dbg = torch.zeros(2 * 128 * 128 + 1024, device='cuda')
lib.psa_debug_set(ctypes.c_void_p(dbg.data_ptr()))
m = np.full((nb, nb), 2)
res = psa.psa_streaming(to_dev(q[0]), pyr, torch.from_numpy(m).cuda())
torch.cuda.synchronize()
S = dbg[:2*128*128].view(2, 128, 128).double().cpu().numpy()
ka = dbg[2*128*128:].view(torch.int32).cpu().numpy()
qt = to_dev(q[0]).double().cpu().numpy()[:128]
kp = pyr.level_k(2)[0, 0].double().cpu().numpy()
ref = qt @ kp[:128].T
print('S[0, 0, :4]', S[0, 0, :4], 'qk', ref[0, :4], 'diff', (S[0] - ref)[0, :4], 'mean diff', (S[0]-ref).mean())
print("ka words", [hex(int(x) & 0xffffffff) for x in ka[:8]])
