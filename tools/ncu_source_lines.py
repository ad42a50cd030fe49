"""Join an ncu source-page capture (SASS, per-instruction metrics) with nvdisasm
line info, aggregating warp instructions / thread instructions / stall samples
per source line of one kernel.

  python tools/ncu_source_lines.py <lib.so> <report.ncu-rep> <mangled-name-fragment> <out.tsv>

NCU_CUBIN selects the cubin (default "march"), NCU_KERNEL the report's kernel
block by a substring of its demangled name (default: the mangled fragment's
base name; set it when several instantiations were captured).
"""
import csv, re, sys, collections, subprocess, os, glob
lib, rep, fn = sys.argv[1], sys.argv[2], sys.argv[3]
d = f"/tmp/cmp/{os.path.basename(lib)}"
os.makedirs(d, exist_ok=True)
subprocess.run(f"cd {d} && cuobjdump -xelf all {lib} >/dev/null 2>&1", shell=True)
cub = [c for c in glob.glob(d+"/*.cubin") if os.environ.get("NCU_CUBIN", "march") in c][0]
txt = subprocess.run(["nvdisasm","-gi",cub],capture_output=True,text=True).stdout.split("\n")
start=None
for i,l in enumerate(txt):
    if l.startswith("_ZN") and fn in l and l.endswith(":"): start=i;break
insts=[];cur=None;prev=False
for l in txt[start+1:]:
    if l.startswith("\t.section") or l.startswith("//----"): break
    m=re.match(r'\s*//## File "([^"]+)", line (\d+)(.*)',l)
    if m and prev: continue
    prev=bool(m)
    if m:
        chain=[(m.group(1).split("/")[-1],int(m.group(2)))]+[(a.split("/")[-1],int(b)) for a,b in re.findall(r'inlined at "([^"]+)", line (\d+)', m.group(3))]
        cur=(chain[0][0],chain[0][1],tuple(chain)); continue
    m=re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*)',l)
    if m: insts.append((m.group(2).strip(),cur))
csvtxt = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source=sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(csvtxt.splitlines()))
# the source page lists one block per profiled kernel: '"Kernel Name",<name>' then a header row
blocks=[]
for i,r in enumerate(rows):
    if r and r[0]=="Kernel Name": blocks.append(i)
blocks.append(len(rows))
sel=None
for bi in range(len(blocks)-1):
    name=rows[blocks[bi]][1] if len(rows[blocks[bi]])>1 else ""
    plain=os.environ.get("NCU_KERNEL", fn.split("ILi")[0])  # e.g. "dt_rmq_kernel<2,"
    if plain in name.replace(" ","") or plain in name:
        sel=(blocks[bi],blocks[bi+1]); break
if sel is None: sel=(blocks[0],blocks[1])
hdr=rows[sel[0]+1];data=rows[sel[0]+2:sel[1]]
iE=hdr.index("Instructions Executed");iT=hdr.index("Thread Instructions Executed");iS=hdr.index("Warp Stall Sampling (All Samples)")
print("rows",len(data),"sass",len(insts))
by=collections.defaultdict(lambda:[0,0,0])
for k in range(min(len(data),len(insts))):
    key=insts[k][1] or ("?",0,())
    # label: innermost location, plus the call-site chain (outermost last)
    lab=f"{key[0]}:{key[1]}" + ("|" + ">".join(f"{f}:{n}" for f,n in key[2][1:]) if len(key) > 2 and key[2][1:] else "")
    by[lab][0]+=int(data[k][iE] or 0);by[lab][1]+=int(data[k][iT] or 0);by[lab][2]+=int(data[k][iS] or 0)
tot=[sum(v[i] for v in by.values()) for i in range(3)]
print("warp inst %.3fG thread inst %.3fG"%(tot[0]/1e9,tot[1]/1e9))
out=sys.argv[4]
with open(out,"w") as f:
    for lab,v in sorted(by.items(),key=lambda kv:-kv[1][0]):
        f.write(f"{lab}\t{v[0]}\t{v[1]}\t{v[2]}\n")
