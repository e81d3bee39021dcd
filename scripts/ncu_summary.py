import csv, subprocess, sys
def raw(rep):
    out = subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout
    r=list(csv.reader(out.splitlines())); h=r[0]; u=r[1]; v=r[2]
    return {n:(v[i],u[i]) for i,n in enumerate(h)}
def stalls(rep, n=18):
    out = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","cuda,sass"],capture_output=True,text=True).stdout
    rows=list(csv.reader(out.splitlines())); file=None; res=[]
    for r in rows:
        if r and r[0]=="File Path": file=r[1].split('/')[-1]; continue
        if len(r)>4 and r[0].isdigit() and r[2]=='-':
            try: res.append((int(r[4]), file, int(r[0]), r[1].strip()))
            except: pass
    tot=sum(o[0] for o in res) or 1
    return [(s, 100*s/tot, f, l, src) for s,f,l,src in sorted(res, reverse=True)[:n]]
KEYS=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','lts__t_sector_hit_rate.pct','lts__throughput.avg.pct_of_peak_sustained_elapsed','sm__throughput.avg.pct_of_peak_sustained_elapsed','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__grid_size','launch__block_size','launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem']
if __name__=="__main__":
    rep=sys.argv[1]
    d=raw(rep)
    for k in KEYS:
        if k in d: print(f"{k:60s} {d[k][0]} {d[k][1]}")
    for s,p,f,l,src in stalls(rep): print(f"{s:7d} {p:5.1f}% {f}:{l} {src[:90]}")
