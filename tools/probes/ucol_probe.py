import sys, os, torch
sys.path.insert(0, os.getcwd())
import bench
sys.argv=[sys.argv[0]]
args=bench.parse()
imgs=bench._batch_images(args, args.seed, args.batch, torch.device("cuda"))
print("batch", imgs.shape)
tot_nw=tot_u=0
for k in range(0, imgs.shape[0], 256):
    t=imgs[k].view(-1,3).to(torch.int64)
    key=t[:,0]|(t[:,1]<<8)|(t[:,2]<<16)
    nw=(t.min(dim=1).values < 220) if False else ~((t >= 220).all(dim=1))
    kk=key[nw][:100000]
    u=torch.unique(kk).numel()
    print(k, int(nw.sum()), kk.numel(), u)
