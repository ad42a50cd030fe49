#!/bin/bash
# Register / spill report of every march_kernel instantiation (ptxas -v), demangled.
# usage: tools/ptxas_report.sh [extra nvcc flags...]
cd "$(dirname "$0")/../paper_2407_10482_b200"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -Xcompiler -ffp-contract=off -I../include -Icsrc --expt-relaxed-constexpr \
  -fmad=false -Xptxas -v "$@" -c csrc/march.cu -o /tmp/march_report.o 2>&1 |
python3 -c '
import re, subprocess, sys
cur = None
spill = ("?", "?")
for line in sys.stdin:
    m = re.search(r"Compiling entry function .(_Z\w+).", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur: spill = (m.group(1), m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur and "march_kernel" in cur:
        t = re.search(r"march_kernel<(.*)>", cur).group(1)
        print(f"march_kernel<{t}>: {m.group(1)} regs, spill st/ld {spill[0]}/{spill[1]}")
        cur = None
'
