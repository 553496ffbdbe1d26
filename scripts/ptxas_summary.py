"""Summarize `nvcc -Xptxas -v` output: kernel, registers, spill bytes, smem."""
import re
import subprocess
import sys

txt = open(sys.argv[1]).read() if len(sys.argv) > 1 else sys.stdin.read()
cur = None
for line in txt.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        name = re.sub(r"sta::\(anonymous namespace\)::", "", name)
        name = re.sub(r"\(.*", "", name)
        cur = name
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        sm = re.search(r"(\d+) bytes smem", line)
        print(f"{cur:50s} regs={m.group(1):>4} smem={sm.group(1) if sm else 0:>6} spill={spill}")
        cur = None
