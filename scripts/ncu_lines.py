"""Samples per CUDA source line from a .ncu-rep (needs -lineinfo + --import-source on)."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
cur_file, H, lines, tot = "?", None, [], 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
    elif len(r) > 6 and r[0] == "Line No":
        H = {h: i for i, h in enumerate(r)}
    elif H and len(r) > 6 and r[0].isdigit():  # a source-line row (SASS rows have an empty line number)
        n = int(r[H["# Samples"]]) if r[H["# Samples"]].isdigit() else 0
        tot += n
        lines.append((n, cur_file, r[0], r[1].strip()[:100], r[H["Instructions Executed"]]))
print("total samples", tot)
for n, f, ln, src, ins in sorted(lines, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{n:6d} {100*n/max(tot,1):5.1f}% inst {ins:>10s} {f}:{ln:>4s}  {src}")
