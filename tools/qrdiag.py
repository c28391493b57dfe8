import sys, time, numpy as np
sys.path.insert(0,'.')
import paper_1703_09074_b200 as rcp
ctx = rcp.default_context()
rng = np.random.default_rng(0)
for (I,n) in [(400,30),(1024,70),(128,48)]:
    for cond in [1e1, 1e3, 1e5]:
        m = rng.standard_normal((I,n)) @ np.diag(np.logspace(0, -np.log10(cond), n)) @ rng.standard_normal((n,n))
        m = np.asfortranarray(m)
        rcp.thin_qr(m)
        t0=time.perf_counter()
        for _ in range(20): q, rw = rcp.thin_qr(m)
        dt=(time.perf_counter()-t0)/20*1e6
        names=[p[0] for p in ctx.pass_timings()]
        print(I, n, 'cond~%.0e'%np.linalg.cond(m), 'us/call(host)', round(dt,1))
