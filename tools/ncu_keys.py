import csv,sys,json
keys=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','lts__t_sector_hit_rate.pct','l1tex__t_sector_hit_rate.pct','sm__throughput.avg.pct_of_peak_sustained_elapsed','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__grid_size','launch__block_size','lts__throughput.avg.pct_of_peak_sustained_elapsed','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__cycles_elapsed.avg.per_second','l1tex__m_xbar2l1tex_read_bytes.sum']
out={}
for f in sys.argv[1:]:
    rows=list(csv.reader(open(f))); hdr,units=rows[0],rows[1]
    for r in rows[2:]:
        d={}
        for k in keys:
            if k in hdr:
                i=hdr.index(k); d[k]=r[i]+' '+units[i]
        st={h[len('smsp__pcsamp_warps_issue_stalled_'):]:float(r[i].replace(',','')) for i,h in enumerate(hdr) if h.startswith('smsp__pcsamp_warps_issue_stalled_') and not h.endswith('not_issued')}
        tot=sum(st.values()) or 1
        d['top_stalls_pct']={k:round(100*v/tot,1) for k,v in sorted(st.items(), key=lambda kv:-kv[1])[:5]}
        out[f.split('/')[-1]+' :: '+r[hdr.index('Kernel Name')].split('(')[0]]=d
print(json.dumps(out,indent=1))
