# key metrics of every kernel in an ncu report: tools/ncu_sum.sh report.ncu-rep
ncu -i "$1" --page raw --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,launch__grid_size 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
cols=[i for i in range(len(h)) if '__' in h[i]]
for row in r[2:]:
    print(row[h.index('Kernel Name')][:48].ljust(48), ' '.join(h[i].split('__')[1].split('.')[0][:14]+'='+row[i] for i in cols))
"
