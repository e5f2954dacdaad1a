import numpy as np, torch, sys
sys.path.insert(0, '.')
from tests.test_gpu_batched import _corr_exact
for (K,N,B) in [(128,128,128),(384,256,256)]:
    rng = np.random.default_rng(K + N + B)
    D = rng.standard_normal((K, N))
    V = rng.standard_normal((B, N))
    Dt = torch.from_numpy(D).to(torch.bfloat16).cuda()
    out = _corr_exact(Dt, torch.from_numpy(V).cuda()).cpu().numpy()
    Dh = Dt.double().cpu().numpy()
    ref = V @ Dh.T
    err = np.abs(out-ref); bound = np.abs(V) @ np.abs(Dh).T
    r = err/bound
    print(K,N,B, 'max rel', r.max(), 'median', np.median(r))
    print(' out[0,:4]', out[0,:4]); print(' ref[0,:4]', ref[0,:4])
    bad = np.argwhere(r > 1e-6)
    print(' nbad', len(bad), bad[:5])
    if len(bad):
        rows = np.unique(bad[:,0]); cols=np.unique(bad[:,1]); print(' rows', rows[:20], len(rows), 'cols', cols[:20], len(cols))
        print(' ratio out/ref', (out[bad[:5,0],bad[:5,1]]/ref[bad[:5,0],bad[:5,1]]))
