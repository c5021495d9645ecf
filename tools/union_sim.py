"""CPU model of the force sweep's work split (test-side tool, uses the oracle IC): for a
uniform box at ppc 1024 it rebuilds the kernel's spatial order (8x8 sub-cell Morton bins per
cell, stable), 32-particle j chunks, the warp-box/reach near test, and counts, for warps of
32 / 16 / 8 particles (1 / 2 / 4 lanes per particle): the share of near chunks, the share of
pair-column iterations whose SPH block runs (any lane in support), and the lane slots spent
per in-support pair. Reproduces the ncu numbers of force2_kernel (near 47 %, blocks on 65 %
of near columns, 72 % lane use) and bounds what smaller i-boxes could save.
    python tools/union_sim.py
"""
import sys, numpy as np
sys.path.insert(0, '/root/repo')
from oracle import Oracle
orc = Oracle()
n, ppc = 147456, 1024   # nx = 12
recs, par = orc.make_particles(n, ppc, 42)
nx = orc.grid_nx(n, ppc); ny = nx
x = recs['x'].copy(); h = recs['h'].copy()
cell = np.minimum((x[:,0]*nx).astype(int), nx-1) + nx*np.minimum((x[:,1]*ny).astype(int), ny-1)
# slots in (cell, all) order; ilist: per cell stable sort by Morton bin
order = np.lexsort((np.arange(n), cell))
cx = (order*0); 
def morton(p, c):
    cy, cxx = c // nx, c % nx
    bx = np.clip(np.floor((x[p,0]*nx - cxx)*8).astype(int), 0, 7)
    by = np.clip(np.floor((x[p,1]*ny - cy)*8).astype(int), 0, 7)
    m = np.zeros_like(bx)
    for b in range(3): m |= (((bx>>b)&1)<<(2*b)) | (((by>>b)&1)<<(2*b+1))
    return m
cells = {}
for c in range(nx*ny):
    p = order[cell[order]==c]
    m = morton(p, c)
    cells[c] = p[np.argsort(m, kind='stable')]
rng = np.random.default_rng(1)
def stencil(c):
    cy, cxx = divmod(c, nx)
    out=[]
    for dy in (-1,0,1):
        for dx in (-1,0,1):
            k=((cy+dy)%ny)*nx+(cxx+dx)%nx
            if k not in [o[0] for o in out]: out.append((k, dx, dy))
    return out
def stats(group, js):
    tot_cols=0; exec_cols=0; near_ch=0; all_ch=0; in_pairs=0; lane_slots=0
    for c in [int(v) for v in rng.choice(nx*ny, 12, replace=False)]:
        loc = cells[c]
        for g0 in range(0, len(loc), group):
            I = loc[g0:g0+group]
            xi = x[I]; hi = h[I]; R2 = (2.5*hi)**2
            for (k, dx, dy) in stencil(c):
                J = cells[k]
                xj = x[J] + np.array([0,0])
                # periodic shift
                sh = np.array([0.0,0.0])
                cy, cxx = divmod(c, nx); ky, kx = divmod(k, nx)
                ddx = kx - cxx; ddy = ky - cy
                if ddx > 1: sh[0] = -1.0
                if ddx < -1: sh[0] = 1.0
                if ddy > 1: sh[1] = -1.0
                if ddy < -1: sh[1] = 1.0
                xj = xj + sh
                for ch in range(0, len(J), 32):
                    xc = xj[ch:ch+32]
                    d2 = ((xi[:,None,:]-xc[None,:,:])**2).sum(-1)
                    ins = (d2 < R2[:,None]) & (d2 > 0)
                    all_ch += 1
                    # near if any pair within reach of box (approx: any in support)
                    boxlo = xi.min(0); boxhi = xi.max(0); reach = 2.5*hi.max()
                    gx = np.maximum(0, np.maximum(xc[:,0]-boxhi[0], boxlo[0]-xc[:,0]))
                    gy = np.maximum(0, np.maximum(xc[:,1]-boxhi[1], boxlo[1]-xc[:,1]))
                    cbl = xc.min(0); cbh = xc.max(0)
                    bgx = max(0, max(cbl[0]-boxhi[0], boxlo[0]-cbh[0])); bgy = max(0, max(cbl[1]-boxhi[1], boxlo[1]-cbh[1]))
                    near = bgx*bgx+bgy*bgy <= reach*reach
                    if not near: continue
                    near_ch += 1
                    in_pairs += ins.sum()
                    if js == 1:
                        cols = ins.any(0)          # per j column
                        tot_cols += ins.shape[1]; exec_cols += cols.sum()
                        lane_slots += cols.sum()*32
                    else:
                        # lanes = (i, slice); iteration t covers j = js*t + slice
                        nj = ins.shape[1]
                        for t in range(0, (nj+js-1)//js):
                            js_idx = [js*t+q for q in range(js) if js*t+q < nj]
                            e = ins[:, js_idx].any()
                            tot_cols += 1; exec_cols += e
                            lane_slots += e*32
    return dict(near_frac=near_ch/all_ch, exec_per_iter=exec_cols/max(tot_cols,1), lane_util=in_pairs/max(lane_slots,1), sph_lane_slots_per_inpair=lane_slots/max(in_pairs,1), near_ch=near_ch, iters=tot_cols)
for group, js in ((32,1),(16,2),(8,4)):
    rng = np.random.default_rng(1)
    print(group, js, stats(group, js))
