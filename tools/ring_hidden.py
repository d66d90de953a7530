"""Ring communication hidden fraction from each rank's device
timeline of one pipelined layer: the compute stream's idle time between ring steps is the
exposed part of the transfers,
    hidden = 1 - sum_r max(0, compute_begin[r] - compute_end[r-1]) / sum_r transfer[r],
and the SPEC closed form 1 - (t_pipelined - R t_compute_step) / ((R-1) t_comm_step) beside it.
Ranks are threads sharing ONE GPU here (copy-engine transfers; every rank's compute step
shares the SMs with the other ranks'), so this shows whether the transfers overlap the
compute, not NVLink numbers.  usage: python tools/ring_hidden.py"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_10940_b200 as fu


def one(n, r, heads, s):
    sl = s // n
    q = [torch.empty(1, heads, sl, 128, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(n)]
    k = [torch.empty_like(x).uniform_(-1, 1) for x in q]
    v = [torch.empty_like(x).uniform_(-1, 1) for x in q]
    mesh = fu.make_mesh(n, r)
    opts = fu.CommOptions(pipelined_ring=True, out_dtype=torch.float16, check_finite=False)

    def prog(ctx):
        i = ctx.rank()
        for _ in range(3):
            fu.usp_attention(ctx, q[i], k[i], v[i], mesh, opts)
        torch.cuda.synchronize()
        fu.usp_attention(ctx, q[i], k[i], v[i], mesh, opts)
        torch.cuda.synchronize()
        tl = ctx.timeline()
        comp, comm = ctx.ring_timings()
        return tl, comp, comm

    res = fu.run_protocol(n, prog).results
    out = []
    for rank, (tl, comp, comm) in enumerate(res):
        cb = {e["round"]: e["t_ms"] for e in tl if e["kind"] == "compute_begin"}
        ce = {e["round"]: e["t_ms"] for e in tl if e["kind"] == "compute_end"}
        exposed = sum(max(0.0, cb[i] - ce[i - 1]) for i in range(1, r))
        total_comm = sum(comm[1:])
        t_pipe = ce[r - 1] - min(cb[0], min(e["t_ms"] for e in tl))
        spec = 1.0 - (t_pipe - r * statistics.mean(comp)) / ((r - 1) * statistics.mean(comm[1:]))
        out.append({"rank": rank, "exposed_ms": exposed, "comm_ms": total_comm,
                    "hidden": 1.0 - exposed / total_comm if total_comm > 0 else None,
                    "hidden_spec_formula": spec, "t_pipelined_ms": t_pipe,
                    "compute_ms": comp, "comm_step_ms": comm})
    hid = [o["hidden"] for o in out if o["hidden"] is not None]
    print(json.dumps({"measure": "ring_hidden_fraction", "n_ranks": n, "ulysses": n // r, "ring": r,
                      "seq": s, "heads": heads, "hidden_median": statistics.median(hid),
                      "hidden_min": min(hid),
                      "spec_formula_median": statistics.median(o["hidden_spec_formula"] for o in out),
                      "note": "ranks share one GPU: copy-engine transfers, SMs shared by every rank's compute",
                      "per_rank": out}), flush=True)


for n, r, heads, s in ((2, 2, 12, 8448), (4, 4, 6, 16896), (8, 4, 24, 16896)):
    one(n, r, heads, s)
