"""Marked-pixel fraction of the global pass for several RGB cell geometries
(NumPy estimate on a reference-rendered slide)."""
import numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from oracle import spcn_oracle as orc
W = orc.he_basis()
i0 = np.array([255.,255,255])
lut = orc.od_table(i0)  # (3,256)
g = W.T @ W
det = g[0,0]*g[1,1]-g[0,1]**2
def dens(v):  # v (3,N)
    t = W.T @ v
    u0 = np.maximum(0, (g[1,1]*t[0]-g[0,1]*t[1])/det)
    h1 = np.maximum(0, (t[1]-g[0,1]*u0)/g[1,1])
    h0 = np.maximum(0, (t[0]-g[0,1]*h1)/g[0,0])
    return h0, h1
lo = np.array([1.87, 1.868])
# all colours
c = np.arange(1<<24, dtype=np.int64)
r, gg, b = c & 255, (c>>8)&255, c>>16
h0, h1 = dens(np.stack([lut[0][r], lut[1][gg], lut[2][b]]))
cand = ((h0 >= lo[0]-0.01) | (h1 >= lo[1]-0.01)) & ~((r>220)&(gg>220)&(b>220))
white = (r>220)&(gg>220)&(b>220)
px,_,_ = orc.render(1024, 1024, 3, tissue_fraction=0.6)
px = px.reshape(-1,3).astype(np.int64)
for name,(sr,sg,sb) in {"8x8x8":(3,3,3),"4x4x32":(2,2,5),"4x8x16":(2,3,4),"8x4x16":(3,2,4), "4x4x16(64K)":(2,2,4)}.items():
    cell = (r>>sr) | ((gg>>sg) << (8-sr)) | ((b>>sb) << (16-sr-sg))
    ncell = cell.max()+1
    anyc = np.zeros(ncell,bool); np.logical_or.at(anyc, cell, cand)
    anyw = np.zeros(ncell,bool); np.logical_or.at(anyw, cell, white)
    anynw = np.zeros(ncell,bool); np.logical_or.at(anynw, cell, ~white)
    cls = np.where(anyc|(anyw&anynw), 2, np.where(anynw,1,0))
    pc = (px[:,0]>>sr) | ((px[:,1]>>sg) << (8-sr)) | ((px[:,2]>>sb) << (16-sr-sg))
    k = cls[pc]
    truec = cand[px[:,0] | (px[:,1]<<8) | (px[:,2]<<16)]
    print(name, "cells", ncell, "marked frac %.4f" % (k==2).mean(), "true cand %.4f" % truec.mean())
