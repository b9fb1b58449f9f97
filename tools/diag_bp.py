import numpy as np, torch, sys
sys.path.insert(0, '.')
import oracle, rmx_synth as syn, paper_1403_5524_b200 as rmx
ctx = rmx.Context()
c = syn.make_case("bp", ne=2000)
idx = syn.parity_sample(c, 6, n_pole=2, n_thresh=2)
E = c.E[idx]
F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
no = syn.n_open(c.eps, E)
R, st = ctx.build_R(c.w, c.Ek, c.a, E)
K, st = ctx.match_K(R, F, G, Fp, Gp, c.a, no, status=st)
T2, rs, st = ctx.collision_strength(K, no, status=st)
torch.cuda.synchronize()
K = K.cpu().numpy(); R = R.cpu().numpy(); T2 = T2.cpu().numpy()
ref = oracle.sweep(c.w, c.Ek, c.a, E, F, G, Fp, Gp, no, np.arange(len(idx)), diag=True, threads=16)
for p in range(len(idx)):
    o = no[p]
    A = np.diag(G[p]) - c.a * ref["R"][p] * Gp[p][None, :]
    As = A / np.max(np.abs(A), axis=0)[None, :]
    cs = np.linalg.cond(As, 1)
    # GPU K from oracle R in fp64 numpy (library solve) for comparison
    B = np.diag(F[p]) - c.a * ref["R"][p] * Fp[p][None, :]
    Knp = -np.linalg.solve(A, B[:, :o])
    def nrel(x, r): return float(np.max(np.abs(x - r)) / np.max(np.abs(r)))
    print(f"p={p} E={E[p]:.6f} o={o} cond1(A)={ref['diag'][p,2]:.3e} cond1(Acolscaled)={cs:.3e} "
          f"|K|max={np.max(np.abs(ref['K'][p][:o,:o])):.3e} errK_gpu={nrel(K[p][:o,:o], ref['K'][p][:o,:o]):.3e} "
          f"errK_numpy={nrel(Knp[:o,:o], ref['K'][p][:o,:o]):.3e} errR={nrel(R[p], ref['R'][p]):.2e} errT2={nrel(T2[p], ref['T2'][p]):.2e} asymK={ref['diag'][p,1]:.2e}")
print("--- GPU match from oracle R; numpy solve from GPU R")
Ko, _ = ctx.match_K(torch.from_numpy(ref["R"]), F, G, Fp, Gp, c.a, no)
Ko = Ko.cpu().numpy()
for p in range(len(idx)):
    o = no[p]
    A = np.diag(G[p]) - c.a * R[p] * Gp[p][None, :]
    B = np.diag(F[p]) - c.a * R[p] * Fp[p][None, :]
    Knp = -np.linalg.solve(A, B[:, :o])
    def nrel(x, r): return float(np.max(np.abs(x - r)) / np.max(np.abs(r)))
    print(f"p={p} errK_gpu(oracleR)={nrel(Ko[p][:o,:o], ref['K'][p][:o,:o]):.3e} errK_numpy(gpuR)={nrel(Knp[:o,:o], ref['K'][p][:o,:o]):.3e}")
