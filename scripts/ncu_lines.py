"""Instructions executed and stall samples per CUDA source line, from a .ncu-rep (needs -lineinfo): where the warp-instructions go."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
cur, hdr, out = "?", None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
    elif hdr and r[0].isdigit():
        try:
            out.append((int(r[hdr["Instructions Executed"]]), int(r[hdr["# Samples"]]), cur, int(r[0]), r[1].strip()))
        except Exception:
            pass
tot = sum(o[0] for o in out) or 1
stot = sum(o[1] for o in out) or 1
print(f"total warp-instructions {tot}, samples {stot}")
byfile = {}
for n, s, f, ln, src in out:
    a = byfile.setdefault(f, [0, 0])
    a[0] += n; a[1] += s
for f, (n, s) in sorted(byfile.items(), key=lambda kv: -kv[1][0]):
    print(f"  {f:22s} {100 * n / tot:5.1f}% instr  {100 * s / stot:5.1f}% samples")
for n, s, f, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{100 * n / tot:5.1f}% {100 * s / stot:5.1f}%s {f}:{ln:<4d} {src[:110]}")
