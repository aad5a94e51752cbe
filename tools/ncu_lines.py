"""Per-CUDA-line stall samples / instructions from an ncu report (needs -lineinfo).

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = "?"
hdr = None
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0] or r[0] in ("Function Name",):
        continue
    try:
        samples = int(r[4])
        inst = int(r[7])
    except (ValueError, IndexError):
        continue
    stalls = {hdr[i][6:]: int(r[i]) for i in range(len(hdr)) if hdr[i].startswith("stall_")
              and "Not Issued" not in hdr[i] and r[i].isdigit() and int(r[i]) > 0}
    rows.append((samples, inst, fname, int(r[0]), r[1].strip()[:70], stalls))
S = sum(x[0] for x in rows)
I = sum(x[1] for x in rows)
print(f"total samples {S}  warp instructions {I}")
for s, i, f, ln, src, st in sorted(rows, reverse=True)[:top]:
    tops = ", ".join(f"{k}:{100 * v / max(s, 1):.0f}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
    print(f"{100 * s / S:5.1f}% {100 * i / I:5.1f}%i {f}:{ln:<4d} {src:70s} [{tops}]")
