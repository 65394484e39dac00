"""SASS instructions per source line of one kernel in librs.so (code-size
profile: the warp-leaf kernels are partly instruction-fetch bound).
    python tools/sass_lines.py k_leaf_warp_wor_tu_p2 [top]"""
import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
kern, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_1610_05141_b200", "librs.so")],
                   cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
lines = sass.split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith("//--------------------- .text.") and kern + "ENS_" in l)
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith("//--------------------- .text.")), len(lines))
cur, cnt = None, collections.Counter()
for l in lines[start:end]:
    m = re.search(r'## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        cnt[cur] += 1
print("total", sum(cnt.values()))
srcs = {}
for (k, v) in cnt.most_common(top):
    txt = ""
    if k and os.path.exists(os.path.join(ROOT, "paper_1610_05141_b200", "csrc", k[0])):
        srcs.setdefault(k[0], open(os.path.join(ROOT, "paper_1610_05141_b200", "csrc", k[0])).read().split("\n"))
        txt = srcs[k[0]][k[1] - 1].strip()[:110]
    print(f"{v:5d} {k[0] if k else '?'}:{k[1] if k else 0}  {txt}")
