"""Static SASS census of a kernel's hottest loop (the walk-step loop).

    python tools/sass_loop.py [kernel-substring]

Disassembles libsokol.so with line info (nvdisasm), finds the largest
backward branch region of the named kernel and prints its instruction count,
opcode histogram and per-source-line counts.  Used to check a change's
effect on the per-step instruction budget before spending GPU time.
"""
import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
name = sys.argv[1] if len(sys.argv) > 1 else "saw_walk_kernelILi2ELb0ENS_8EvalFastILi1ELi10EEELi4"
lib = os.environ.get("SOKOL_LIB") or os.path.join(ROOT, "paper_2210_15962_b200", "libsokol.so")
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(d, cub)], capture_output=True, text=True).stdout
sym = name if name.startswith("_") else (f"_ZN2sk15{name}" if name.startswith("saw_walk") else f"_ZN2sk{len(name.split('I')[0])}{name}")
start = re.search(r"\n\.text\." + re.escape(sym) + r"[^:\n]*:", txt).start()
body = txt[start:]
nxt = body.find("\n.text.", 10)
body = body[: nxt if nxt > 0 else None]
cur, ins = None, []
labels = {}
for ln in body.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"^(\.L_x_\d+):", ln)
    if m:
        labels[m.group(1)] = len(ins)
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip(), cur))
best = None
key_op = sys.argv[2] if len(sys.argv) > 2 else "HMMA"  # the step loop: smallest loop containing this opcode
for i, (a, t, _) in enumerate(ins):
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?`\((\.L_x_\d+)\)", t)
    if m and m.group(1) in labels and labels[m.group(1)] < i:
        j0 = labels[m.group(1)]
        if not any(key_op in x[1] for x in ins[j0: i + 1]):
            continue
        if best is None or i - j0 < best[1] - best[0]:
            best = (j0, i)
lo, hi = best
loop = ins[lo: hi + 1]
print(f"loop: {len(loop)} static instructions ({hex(loop[0][0])}..{hex(loop[-1][0])})")
ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for _, t, _ in loop)
print("opcodes:", ", ".join(f"{k}={v}" for k, v in ops.most_common(18)))
lines = collections.Counter(f"{s[0]}:{s[1]}" for _, _, s in loop if s)
print("top lines:", ", ".join(f"{k}={v}" for k, v in lines.most_common(25)))
if os.environ.get("SASS_DUMP"):
    with open(os.environ["SASS_DUMP"], "w") as f:
        for a, t, s in loop:
            f.write(f"{a:05x}  {t:70s}  {s[0] + ':' + str(s[1]) if s else ''}\n")
