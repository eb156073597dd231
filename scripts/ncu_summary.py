"""Headline metrics + stall mix + top source lines of one kernel in an ncu report.
usage: python scripts/ncu_summary.py report.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)))
d = dict(zip(raw[0], raw[2]))
keys = ["gpu__time_duration.sum", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.avg.per_cycle_active", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]
for k in keys:
    print("%-100s %s %s" % (k, d.get(k, "?"), raw[1][raw[0].index(k)] if k in raw[0] else ""))
st = sorted(((float(v), n[34:]) for n, v in d.items() if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued") and v.replace(".", "").isdigit()), reverse=True)
t = sum(x for x, _ in st)
print("stalls: " + " ".join("%s %.1f%%" % (n, 100 * x / t) for x, n in st[:9]))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = []; hdr = None; fname = None
for rec in csv.reader(io.StringIO(out)):
    if not rec: continue
    if rec[0] == "File Path": fname = rec[1].split("/")[-1]; continue
    if rec[0] == "Line No": hdr = rec; continue
    if hdr is None or rec[0] == "": continue
    dd = dict(zip(hdr, rec))
    iv = lambda k: int(dd.get(k, "0")) if dd.get(k, "0").isdigit() else 0
    rows.append((iv("Instructions Executed"), iv("Warp Stall Sampling (All Samples)"), fname, rec[0], rec[1][:90].strip()))
ti = sum(r[0] for r in rows) or 1; ts = sum(r[1] for r in rows) or 1
print("total warp instructions %d" % ti)
print(" instr  stall  line")
for r in sorted(rows, key=lambda r: -r[1])[:top]:
    print("%5.2f%% %5.2f%%  %s:%s  %s" % (100 * r[0] / ti, 100 * r[1] / ts, r[2], r[3], r[4]))
