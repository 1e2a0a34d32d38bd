"""Summarise an .ncu-rep (element / face kernels): key metrics per launch, stall-sampled source
lines, shared wavefronts per opcode.   python tools/ncu_summary.py rep.ncu-rep [nlines]"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_barrier",
        "smsp__pcsamp_warps_issue_stalled_mio_throttle", "smsp__pcsamp_warps_issue_stalled_lg_throttle",
        "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
        "smsp__pcsamp_warps_issue_stalled_not_selected", "smsp__pcsamp_warps_issue_stalled_selected",
        "smsp__pcsamp_warps_issue_stalled_dispatch_stall", "smsp__pcsamp_warps_issue_stalled_membar",
        "smsp__pcsamp_warps_issue_stalled_no_instructions", "smsp__pcsamp_warps_issue_stalled_branch_resolving",
        "smsp__pcsamp_warps_issue_stalled_drain", "smsp__pcsamp_warps_issue_stalled_imc_miss",
        "smsp__pcsamp_warps_issue_stalled_tex_throttle", "smsp__pcsamp_warps_issue_stalled_sleeping",
        "smsp__pcsamp_warps_issue_stalled_misc"]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    nl = int(sys.argv[2]) if len(sys.argv) > 2 else 14
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr = raw[0]
    for row in raw[2:]:
        d = dict(zip(hdr, row))
        print(d.get("Kernel Name", "?")[:90])
        for k in KEYS:
            if k in d and d[k] not in ("", "0"):
                print(f"   {k} = {d[k]}")
    src = run([rep, "--page", "source", "--csv", "--print-source", "sass"]) if False else ""
    out = run([rep, "--page", "source", "--csv"])
    launch = -1
    rows = []
    hdr = None
    for line in csv.reader(io.StringIO(out)):
        if not line:
            continue
        if line[0].startswith("Kernel Name") or (len(line) == 1 and "opV" in line[0]):
            continue
        if "Source" in line and "Address" in line:
            if rows:
                report(rows, hdr, launch, nl)
            hdr = line
            rows = []
            launch += 1
            continue
        if hdr and len(line) == len(hdr):
            rows.append(line)
    if rows:
        report(rows, hdr, launch, nl)


def report(rows, hdr, launch, nl):
    def col(name):
        for i, h in enumerate(hdr):
            if h.strip().startswith(name):
                return i
        return None

    ci = col("Warp Stall Sampling (All")
    si = col("Source")
    op = col("Instruction") 
    if ci is None:
        print("columns:", hdr)
        return
    ex = lambda name: hdr.index(name) if name in hdr else None
    wi, ii, ei = ex("L1 Wavefronts Shared"), ex("L1 Wavefronts Shared Ideal"), ex("Instructions Executed")
    ops = {}
    if wi is not None:
        for r in rows:
            w = float(r[wi] or 0)
            if w <= 0:
                continue
            toks = r[si].replace("@P0", "").replace("@!P0", "").split()
            op = next((t for t in toks if t[:3] in ("LDS", "STS", "LDG", "ATO", "RED")), toks[0] if toks else "?")
            o = ops.setdefault(op, [0.0, 0.0, 0.0])
            o[0] += w
            o[1] += float(r[ii] or 0)
            o[2] += float(r[ei] or 0)
    tot = sum(float(r[ci] or 0) for r in rows)
    print(f"--- launch {launch}: stall samples {tot:.0f}")
    if ops:
        print(f"--- launch {launch}: shared wavefronts by opcode")
        for op, (w, i, n) in sorted(ops.items(), key=lambda kv: -kv[1][0]):
            print(f"  {op:<26} wavefronts {w:>10.0f} ideal {i:>10.0f} inst {n:>10.0f}")
    best = sorted(rows, key=lambda r: -float(r[ci] or 0))[:nl]
    for r in best:
        ls = col("stall_long_sb"); ss = col("stall_short_sb"); bs = col("stall_barrier")
        print(f" {100 * float(r[ci] or 0) / max(tot, 1):5.1f}%  long {r[ls]:>5} short {r[ss]:>5} bar {r[bs]:>5}  {r[si][:130]}")


if __name__ == "__main__":
    main()
