import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle.ddh_oracle as O, synth
from test_gpu_parity import frames, gpu_kwargs, oracle_params, phi_err, r_err
from paper_2305_03284_b200 import DDH
DEV = torch.device("cuda:0")
n, S = 64, 1
for diam in (64, 50, 60, 63):
  for rs, ps, tt in [(0.5, 0.5, True), (0.0, 0.0, True), (0.5, 0.5, False), (0.0, 0.0, False)]:
    p = oracle_params(n, diam=diam, noise_var=0.15, r_sigma=rs, phi_sigma=ps, tiptilt=tt)
    y, ph, c = frames(n, S, 3)
    a = O.aperture_of(p)
    for init in ("cold", "boot"):
        if init == "boot":
            r0, phi0, _ = O.bootstrap(y[0, 0], p, 8, a)
        else:
            r0, phi0 = np.full((n, n), 1e-4), np.zeros((n, n))
        r32, p32 = r0.astype(np.float32), phi0.astype(np.float32)
        ctx = DDH(n, S, aperture_diam=diam, **gpu_kwargs(p))
        ctx.set_state(torch.from_numpy(r32[None]).to(DEV), torch.from_numpy(p32[None]).to(DEV), 1)
        po = torch.empty((1, S, n, n), device=DEV); ro = torch.empty_like(po)
        ctx.step(torch.from_numpy(y[1:2]).to(DEV), po, ro)
        rr, pp, _ = O.ddh_step(r32.astype(np.float64), p32.astype(np.float64), y[1, 0], p, a)
        pg = po[0, 0].cpu().numpy(); rg = ro[0, 0].cpu().numpy()
        d = np.abs(np.angle(np.exp(1j * (pg - pp))))
        print(f"D={diam} r_sig={rs} phi_sig={ps} tiptilt={tt} {init}: phi_err={phi_err(pg, pp, a):.3e} "
              f"r_err={r_err(rg, rr, np.zeros((n,n),bool)):.3e} maxd_in={d[a>0].max():.3e} maxd_out={d[a==0].max() if (a==0).any() else 0:.3e} "
              f"argmax={np.unravel_index(np.argmax(d*(a>0)), d.shape)}")
