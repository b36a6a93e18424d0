"""Key launch / occupancy / stall metrics of every kernel in an ncu report (--page raw).
usage: python tools/ncu_quick.py report.ncu-rep"""
import csv,sys,subprocess,io
rep=sys.argv[1]
raw=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
rows=list(csv.reader(io.StringIO(raw)))
hdr=rows[0]
want=['gpu__time_duration.sum','sm__cycles_active.avg','sm__cycles_active.max','smsp__inst_executed.sum','launch__grid_size','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active','launch__shared_mem_per_block_dynamic','launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem']
for r in rows[2:]:
    d=dict(zip(hdr,r))
    print(d['Kernel Name'][:50])
    for k in want:
        if k in d: print('  ',k,d[k])
    st={k.replace('smsp__pcsamp_warps_issue_stalled_',''):d[k] for k in hdr if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('not_issued')}
    st={k:int(v) for k,v in st.items() if v and v!='0'}
    print('   stalls',sorted(st.items(),key=lambda x:-x[1])[:10])
