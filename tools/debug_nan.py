import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2602_10940_b200 as fu
from oracle.make_golden import qkv
from oracle import restate as R
for (b,h,sq,skv) in [(1,2,200,130),(1,1,128,128),(1,1,128,130),(1,1,128,256),(1,1,128,250),(1,1,256,129)]:
    q,k,v = qkv((b,h,sq,128),(b,h,skv,128))
    r = fu.attention_with_lse(*(torch.from_numpy(x).cuda().bfloat16() for x in (q,k,v)))
    o = r.out.cpu().numpy(); l = r.lse.cpu().numpy()
    ro, rl = R.attention_with_lse(q,k,v)
    bad = np.argwhere(~np.isfinite(o))
    print((b,h,sq,skv), "nan rows:", np.unique(bad[:,2])[:20] if len(bad) else None, "lse nan:", np.argwhere(~np.isfinite(l))[:5].tolist(),
          "rel", np.linalg.norm(np.nan_to_num(o)-ro)/np.linalg.norm(ro), "lsediff", np.nanmax(np.abs(l-rl)))
