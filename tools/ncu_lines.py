"""Per-source-line instruction and stall shares of one ncu --set full capture
(needs --import-source on and -lineinfo builds).

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [--per UNITS] [--top N] [--kernel IDX]

--per divides the executed warp-instruction counts (e.g. warp-rows of the
k-means kernels: iterations * rows / 32) so lines read as "instructions per unit".
"""
import argparse
import collections
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--per", type=float, default=1.0)
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--launch", type=int, default=None, help="only the N-th captured launch (0-based)")
    ap.add_argument("--by-stall", action="store_true", help="order lines by stall samples")
    args = ap.parse_args()
    cmd = ["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if args.launch is not None:
        cmd += ["--launch-skip", str(args.launch), "--launch-count", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
    ops = collections.Counter()
    cur_file = cur_line = cur_src = None
    hdr = None
    for r in rows:
        if len(r) == 2 and r[0] in ("File Path", "File Name", "Function Name"):
            if r[0] != "Function Name":
                cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        if r[0] != "":
            cur_line, cur_src = int(r[0]), r[1]
            continue
        try:
            n = float(r[hdr.index("Instructions Executed")] or 0)
            w = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        k = (cur_file, cur_line)
        agg[k][0] += n
        agg[k][1] += w
        agg[k][2] = cur_src
        op = r[3].strip().split()
        if op:
            o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
            ops[o.split(".")[0]] += n
    tot = sum(v[0] for v in agg.values()) or 1.0
    totw = sum(v[1] for v in agg.values()) or 1.0
    print(f"total warp instructions {tot:.4g} ({tot / args.per:.1f} per unit)")
    print("opcodes:", ", ".join(f"{o} {n / args.per:.1f}" for o, n in ops.most_common(16)))
    key = (lambda kv: -kv[1][1]) if args.by_stall else (lambda kv: -kv[1][0])
    for k, v in sorted(agg.items(), key=key)[: args.top]:
        print(f"{v[0] / args.per:8.1f} {100 * v[1] / totw:5.1f}%stall  {k[0]}:{k[1]}  {v[2].strip()[:90]}")


if __name__ == "__main__":
    main()
