"""(The key-folded U is dumped in the u_quad_base layout of gala_kernels.cuh since round 2; reorder
before comparing.)  Compare the key-folded kernel's U with the split pair's U + P Cacc (GALA_DEBUG_DUMP).  Runs one layer
twice in subprocesses (GALA_FC_KF=1 / 0) on the same seeded inputs and reports where they differ."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n, L, T, B = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (32, 1, 2, 17)))
code = f"""
import sys; sys.path.insert(0, {ROOT!r}); sys.path.insert(0, {ROOT!r} + '/tests')
import numpy as np, torch
from twins import Twin
tw = Twin({n}, {L}, seed=3)
b, steps = tw.gpu.bsgs_steps({T})
tw.keys_for(steps)
pts2 = tw.gpu.encode_gala_weights(tw.slots({T}), b)
wcan = tw.gpu.fc_tc_weights(pts2, {T}, b)
cts = torch.stack([tw.encrypt(tw.slots())[0] for _ in range({B})])
d_r = tw.gpu.to_device_u32(tw.slots({B}))
tw.gpu.mv_gala2_batch(cts, pts2, {T}, d_r, b, wcan=wcan)
torch.cuda.synchronize()
print('PRIMES', ','.join(str(int(q)) for q in tw.gpu.bfv.all_primes), tw.N)
"""
for kf in ("1", "0"):
    env = dict(os.environ, GALA_FC_KF=kf, GALA_DEBUG_DUMP=f"/tmp/kfdbg{kf}")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    line = [x for x in out.stdout.splitlines() if x.startswith('PRIMES')]
    if not line:
        print(out.stdout[-2000:], out.stderr[-2000:])
        sys.exit(1)
    primes = [int(x) for x in line[0].split()[1].split(',')]
    N = int(line[0].split()[2])
Un = np.fromfile("/tmp/kfdbg1_U.bin", np.uint64)
Uo = np.fromfile("/tmp/kfdbg0_U.bin", np.uint64)
Co = np.fromfile("/tmp/kfdbg0_C.bin", np.uint64)
print("sizes", Un.size, Uo.size, Co.size)
M = L + 1
G = Un.size // (B * 2 * M * N)
print("G", G, "primes", primes)
Un = Un.reshape(B, G, 2, M, N)
Uo = Uo.reshape(B, G, 2, M, N)
Co = Co.reshape(B, G, 2, L, N)
if primes:
    P = primes[L]
    want = Uo.copy()
    for j in range(L):
        q = primes[j]
        want[:, :, :, j, :] = ((Uo[:, :, :, j, :].astype(object) + (P % q) * Co[:, :, :, j, :].astype(object)) % q).astype(np.uint64)
    bad = want != Un
    print("mismatches", int(bad.sum()), "of", bad.size)
    if bad.any():
        idx = np.argwhere(bad)
        print("by input", np.unique(idx[:, 0], return_counts=True))
        print("by group", np.unique(idx[:, 1], return_counts=True))
        print("by comp", np.unique(idx[:, 2], return_counts=True))
        print("by prime", np.unique(idx[:, 3], return_counts=True))
        print("first", idx[:5], Un[tuple(idx[0])], want[tuple(idx[0])])
