import csv, re, subprocess, sys
from collections import Counter, defaultdict
def raw(rep):
    out = subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout
    rows=list(csv.reader(out.splitlines())); return dict(zip(rows[0], rows[2]))
def src(rep):
    out = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
    rows=list(csv.reader(out.splitlines())); return rows[1], rows[2:]
keys=[("gpu__time_duration.sum","duration (ns)"),("launch__registers_per_thread","registers/thread"),
 ("sm__warps_active.avg.pct_of_peak_sustained_active","achieved occupancy %"),
 ("smsp__issue_active.avg.pct_of_peak_sustained_active","issue slots busy %"),
 ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active","XU (MUFU) pipe %"),
 ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active","FMA pipe %"),
 ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active","ALU pipe %"),
 ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active","FP64 pipe %"),
 ("smsp__inst_executed.sum","warp instructions"),
 ("dram__bytes_read.sum","DRAM read"),("dram__bytes_write.sum","DRAM write"),
 ("local_load_bytes","-")]
print("# k_cell on 256 C1 frames (cellbench, round-2 kernels)\n")
print("`ncu --set full --clock-control none --import-source on -k regex:k_cell -s 8 -c 1` (accumulating pass) and `-s 31 -c 1` (final pass) on `variants/cellbench/cellbench_base` (tools/cellbench: 256 synthetic 640x480 frames, the engine's stage sequence to realistic centres, then the two k_cell launches alone).  CUDA-event times of the same binary without ncu: k_cell<ACC> 0.598 ms, final 0.456 ms.\n")
for name, rep in (("k_cell<1,8,1> (association + update)", sys.argv[1]), ("k_cell<0,8,1> (final association)", sys.argv[2])):
    d=raw(rep)
    print(f"## {name}\n")
    print("| metric | value |\n|---|---|")
    for k,lab in keys:
        if k in d: print(f"| {lab} (`{k}`) | {d[k]} |")
    px=78643200
    if "smsp__inst_executed.sum" in d:
        print(f"| warp instructions per pixel x32 | {float(d['smsp__inst_executed.sum'].replace(',',''))*32/px:.1f} |")
    if "dram__bytes_read.sum" in d:
        try:
            tot=float(d["dram__bytes_read.sum"].replace(',',''))+float(d["dram__bytes_write.sum"].replace(',',''))
            print(f"| DRAM bytes per pixel | {tot/px:.2f} (units as reported) |")
        except Exception: pass
    hdr,data=src(rep)
    srci=hdr.index("Source")
    reasons=['stall_not_selected','stall_selected','stall_wait','stall_math','stall_mio','stall_dispatch','stall_short_sb','stall_long_sb','stall_branch_resolving','stall_no_inst']
    idx={r:hdr.index(r) for r in reasons if r in hdr}
    tot=Counter(); byop=defaultdict(Counter)
    for r in data:
        if len(r)<=max(idx.values()): continue
        op=re.sub(r'^@!?U?P\w+\s+','',r[srci].strip()).split()
        if not op: continue
        op=op[0].split('.')[0]
        for k,i in idx.items():
            try: v=int(r[i])
            except: v=0
            tot[k]+=v; byop[k][op]+=v
    T=sum(tot.values())
    print(f"\nWarp-state samples ({T}), share and the opcodes they sit on:\n")
    print("| state | share | top opcodes |\n|---|---|---|")
    for k,v in tot.most_common():
        if v==0: continue
        tops=", ".join(f"{op} {c/v*100:.0f}%" for op,c in byop[k].most_common(4))
        print(f"| {k.replace('stall_','')} | {v/T*100:.1f}% | {tops} |")
    print()
