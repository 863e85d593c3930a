exec(open('profiles/pred_path_timing.py').read().split("e0, e1 = torch.cuda.Event(True)")[0])
torch.cuda.synchronize()
ev = [torch.cuda.Event(True) for _ in range(3)]
res = []
for i in range(120):
    ev[0].record()
    pp2 = dec.predict_props(q, rec, pred, append=(kn, kn))
    ev[1].record()
    dec.step(q, props=pp2)
    ev[2].record()
    torch.cuda.synchronize()
    res.append((ev[0].elapsed_time(ev[1]) * 1e3, ev[1].elapsed_time(ev[2]) * 1e3, int((dec.plan_blk > 0).sum().item())))
import numpy as np
a = np.array(res)
print("props us: median %.1f max %.1f | step us: median %.1f p90 %.1f max %.1f | retrieval groups min %d max %d" % (
    np.median(a[:, 0]), a[:, 0].max(), np.median(a[:, 1]), np.percentile(a[:, 1], 90), a[:, 1].max(), a[:, 2].min(), a[:, 2].max()))
slow = np.argsort(-a[:, 1])[:5]
print("slowest steps:", [(int(i), round(a[i, 1], 1), int(a[i, 2])) for i in slow])
