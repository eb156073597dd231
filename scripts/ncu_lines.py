"""Summarise an ncu source page: top CUDA source lines by stall samples and instructions.
usage: python scripts/ncu_lines.py report.ncu-rep [kernel-regex] [N]"""
import csv, io, re, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 2 and sys.argv[2]:
    args += ["-k", "regex:" + sys.argv[2]]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = []; fname = None; hdr = None; cur = None
tot_s = tot_i = 0
for rec in csv.reader(io.StringIO(out)):
    if not rec: continue
    if rec[0] == "File Path": fname = rec[1].split("/")[-1]; continue
    if rec[0] == "Function Name": continue
    if rec[0] == "Line No": hdr = rec; continue
    if hdr is None: continue
    d = dict(zip(hdr, rec))
    if rec[0] != "":
        iv = lambda k: int(d.get(k, "0")) if d.get(k, "0").isdigit() else 0
        cur = [fname, rec[0], rec[1][:90], iv("Warp Stall Sampling (All Samples)"), iv("Instructions Executed")]
        rows.append(cur); tot_s += cur[3]; tot_i += cur[4]
rows.sort(key=lambda r: -r[3])
print("total samples %d, total warp instr %d" % (tot_s, tot_i))
for r in rows[:top]:
    print("%5.1f%% %5.1f%%  %s:%s  %s" % (100.0 * r[3] / max(tot_s, 1), 100.0 * r[4] / max(tot_i, 1), r[0], r[1], r[2].strip()))
