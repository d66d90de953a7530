"""fastusp command line: verify | simulate | cost.

    python -m paper_2602_10940_b200 verify   --workers 4 --max-ring 2 --dims 1x8x256x128 --seed 7
    python -m paper_2602_10940_b200 simulate --workers 8 --max-ring 4 --dims 1x24x4608x128 --pipelined
    python -m paper_2602_10940_b200 cost     --dims 1x24x4608x128 --format csv

Exit codes: 0 success, 1 internal error / failed check, 2 invalid or
infeasible configuration.  Reports are JSON (or CSV for `cost`) carrying the resolved config.
verify/simulate run on the GPU (ranks as threads over the in-process fabric on one device);
they check the distributed layer against single-GPU attention over the full sequence, the
E4M3 codec's round-trip properties and the traffic closed forms -- no CPU fallback.
"""
from __future__ import annotations

import argparse
import csv
import json
import sys


def parse_dims(s: str):
    parts = [int(x) for x in s.lower().split("x")]
    if len(parts) != 4 or min(parts) < 1:
        raise ValueError(f"--dims must be BxHxSxD, got {s!r}")
    return parts


def resolve(args):
    """Validate the configuration (mesh feasibility, divisibility) before running."""
    from . import api
    b, h, s, d = parse_dims(args.dims)
    mesh = api.build_mesh(args.workers, args.max_ring, h)
    if s % args.workers:
        raise ValueError(f"S={s} not divisible by N={args.workers}")
    return (b, h, s, d), mesh


def _inputs(dims, seed):
    import torch
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return [torch.empty(dims, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1, generator=g)
            for _ in range(3)]


def _run_layer(dims, mesh, seed, fp8, pipelined, out_dtype):
    import torch
    from . import api
    q, k, v = _inputs(dims, seed)
    n = mesh.n
    qs, ks, vs = (api.split_sequence(t, n) for t in (q, k, v))
    opts = api.CommOptions(fp8_kv=fp8, pipelined_ring=pipelined, out_dtype=out_dtype)
    rep = api.run_protocol(n, lambda ctx: (api.usp_attention(ctx, qs[ctx.rank()], ks[ctx.rank()],
                                                             vs[ctx.rank()], mesh, opts),
                                           ctx.traffic_log(), ctx.timeline()))
    out = torch.cat([r[0].float() for r in rep.results], dim=2)
    return (q, k, v), out, [r[1] for r in rep.results], [r[2] for r in rep.results]


def cmd_verify(args) -> int:
    import torch
    from . import api, costmodel
    dims, mesh = resolve(args)
    b, h, s, d = dims
    report = {"command": "verify", "config": vars(args), "mesh": mesh.to_json(), "cases": []}
    ok = True
    # (1) distributed == single-GPU attention over the full sequence, every feasible R
    for r in [x for x in range(1, mesh.n + 1) if mesh.n % x == 0 and h % (mesh.n // x) == 0]:
        m = api.make_mesh(mesh.n, r)
        for pip in (False, True):
            (q, k, v), out, traffic, _ = _run_layer(dims, m, args.seed, False, pip, torch.float32)
            full = api.attention_with_lse(q, k, v).out
            rel = float((out - full).norm() / full.norm())
            w = costmodel.WorkloadProfile(B=b, H=h, S=s, D=d)
            want_a2a = costmodel.comm_volume_ulysses(w, mesh.n // r, 2, out_width=4, n=mesh.n)
            want_ring = costmodel.comm_volume_ring(w, r, mesh.n // r, 2)
            got_a2a = sum(e["bytes"] for e in traffic[0] if e["op"] == "all_to_all")
            got_ring = sum(e["bytes"] for e in traffic[0] if e["op"] == "send")
            passed = rel <= 1e-3 and got_a2a == want_a2a and got_ring == want_ring
            ok &= passed
            report["cases"].append({"case": f"usp_N{mesh.n}_R{r}_{'pipe' if pip else 'serial'}",
                                    "rel_l2_vs_single_gpu": rel, "a2a_bytes": got_a2a,
                                    "a2a_bytes_closed_form": want_a2a, "ring_bytes": got_ring,
                                    "ring_bytes_closed_form": want_ring, "pass": passed})
    # (2) E4M3 codec: all 254 non-NaN codes round-trip, decode is monotone, NaN codes decode NaN
    codes = torch.arange(256, dtype=torch.uint8, device="cuda")
    vals = api.decode_e4m3(codes)
    finite = torch.tensor([(c & 0x7F) != 0x7F for c in range(256)], device="cuda")
    rt = api.encode_e4m3(vals[finite])
    mono = bool((vals[:127][1:] > vals[:127][:-1]).all())
    codec_ok = bool(torch.equal(rt, codes[finite])) and mono and bool(torch.isnan(vals[~finite]).all())
    ok &= codec_ok
    report["cases"].append({"case": "e4m3_codec_roundtrip", "pass": codec_ok})
    report["pass"] = ok
    _emit(args, report)
    return 0 if ok else 1


def cmd_simulate(args) -> int:
    import torch
    from . import api
    dims, mesh = resolve(args)
    (q, k, v), out, traffic, timeline = _run_layer(dims, mesh, args.seed, args.fp8_kv,
                                                   args.pipelined, torch.float32)
    full = api.attention_with_lse(q, k, v).out
    report = {"command": "simulate", "config": vars(args), "mesh": mesh.to_json(),
              "rel_l2_vs_single_gpu": float((out - full).norm() / full.norm()),
              "traffic": [e for t in traffic for e in t], "timeline": timeline}
    _emit(args, report)
    return 0


def cmd_cost(args) -> int:
    from . import costmodel
    b, h, s, d = parse_dims(args.dims)
    hw = costmodel.load_profile(args.hw)
    w = costmodel.WorkloadProfile(B=b, H=h, S=s, D=d, layers=args.layers)
    rows = costmodel.sweep(hw, w, ns=[int(x) for x in args.sweep.split(",")], fp8=args.fp8_kv,
                           compiled=args.compiled)
    if args.format == "csv":
        out = open(args.out, "w", newline="") if args.out else sys.stdout
        wr = csv.DictWriter(out, fieldnames=list(rows[0].keys()))
        wr.writeheader()
        wr.writerows(rows)
        if args.out:
            out.close()
    else:
        _emit(args, {"command": "cost", "config": vars(args), "rows": rows})
    return 0


def _emit(args, report):
    text = json.dumps(report, indent=1, default=str)
    if getattr(args, "out", None):
        with open(args.out, "w") as f:
            f.write(text + "\n")
    else:
        print(text)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2602_10940_b200")
    ap.add_argument("command", choices=["verify", "simulate", "cost"])
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--max-ring", type=int, default=1)
    ap.add_argument("--dims", default="1x24x4608x128")
    ap.add_argument("--fp8-kv", action="store_true")
    ap.add_argument("--pipelined", action="store_true")
    ap.add_argument("--compiled", action="store_true", default=True)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--hw", default=None)
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--sweep", default="1,2,4,8")
    ap.add_argument("--out", default=None)
    ap.add_argument("--format", choices=["json", "csv"], default="json")
    args = ap.parse_args(argv)
    try:
        if args.command == "cost":
            return cmd_cost(args)
        try:
            resolve(args)
        except Exception as e:  # noqa: BLE001 -- infeasible config: exit 2
            print(f"invalid configuration: {e}", file=sys.stderr)
            return 2
        return {"verify": cmd_verify, "simulate": cmd_simulate}[args.command](args)
    except ValueError as e:
        print(f"invalid configuration: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001
        print(f"internal error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
