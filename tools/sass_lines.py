"""Static SASS instruction count per source line of one kernel (nvdisasm --print-line-info):
python tools/sass_lines.py file.cubin kernel_substring [n_top]"""
import re
import subprocess
import sys

cub, kern = sys.argv[1], sys.argv[2]
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["nvdisasm", "--print-line-info", cub], capture_output=True, text=True).stdout
sec = None
cur = None
cnt = {}
ops = {}
for ln in txt.splitlines():
    m = re.match(r"//-+ \.text\.(\S+)", ln)
    if m:
        sec = m.group(1)
        continue
    if sec is None or kern not in sec:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", ln)
    if m and cur:
        cnt[cur] = cnt.get(cur, 0) + 1
        op = m.group(2).split(".")[0]
        ops[op] = ops.get(op, 0) + 1
tot = sum(cnt.values())
print("total", tot)
for (f, l), c in sorted(cnt.items(), key=lambda t: -t[1])[:ntop]:
    print(f"{c:6d}  {f}:{l}")
print("opcodes:", sorted(ops.items(), key=lambda t: -t[1])[:25])
