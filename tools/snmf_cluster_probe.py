import os, sys
sys.path.insert(0, "/root/repo")
exec(open("/root/repo/tools/fit_table_probe.py").read().split('print("m", m)')[0])
print("m", m)
for cl in (8, 12, 16):
    try:
        print(f"snmf cluster={cl}: {timed(lambda: snmf.snmf_batched(flat, off, lut, cfg, cluster=cl)):.1f} us")
        r = snmf.snmf_batched(flat, off, lut, cfg, cluster=cl)
        print("  basis", r.basis.cpu().numpy().ravel()[:3])
    except Exception as e:
        print(cl, "ERR", e)
