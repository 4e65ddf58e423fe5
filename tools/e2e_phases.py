import sys, os
sys.path.insert(0, '.')
import numpy as np, torch, gen, bench
import paper_2308_07173_b200 as g
dev = torch.device('cuda', 0)
sc, mp, T_true, T0 = gen.config_c3()
map_h = torch.from_numpy(mp).pin_memory(); scan_h = torch.from_numpy(sc).pin_memory()
cov_map_h = torch.empty((mp.shape[0], 6), dtype=torch.float32).pin_memory()
ev = lambda: torch.cuda.Event(enable_timing=True)
cp = torch.cuda.Stream(); es = torch.cuda.Stream()
for it in range(4):
    torch.cuda.synchronize()
    with torch.cuda.stream(es):
        e = [ev() for _ in range(6)]
        e[0].record(es)
        cp.wait_stream(es)
        with torch.cuda.stream(cp):
            sd = scan_h.to(dev, non_blocking=True)
            up = torch.cuda.Event(); up.record(cp)
        md = map_h.to(dev, non_blocking=True)
        e[1].record(es)
        imap = g.build_index(md, 0.5)
        _, _, cm = g.knn_cov_self(imap, 20, 1e-3, with_nbr=True)
        g.attach_cov(imap, cm)
        e[2].record(es)
        cp.wait_stream(es)
        with torch.cuda.stream(cp):
            c0 = ev(); c0.record(cp)
            cov_map_h.copy_(cm, non_blocking=True)
            c1 = ev(); c1.record(cp)
        es.wait_event(up)
        iscan = g.build_index(sd, 0.0)
        _, _, cs = g.knn_cov_self(iscan, 20, 1e-3, with_nbr=True)
        e[3].record(es)
        T, info = g.align(sd, cs, imap, cm, T0)
        e[4].record(es)
        es.wait_stream(cp)
        e[5].record(es)
    torch.cuda.synchronize()
    print("h2d map %.3f | map build+knn %.3f | scan %.3f | align %.3f | wait d2h %.3f | total %.3f | d2h copy %.3f (starts %.3f after e0)" % (
        e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3]), e[3].elapsed_time(e[4]), e[4].elapsed_time(e[5]), e[0].elapsed_time(e[5]), c0.elapsed_time(c1), e[0].elapsed_time(c0)))
    imap.free(); iscan.free()
