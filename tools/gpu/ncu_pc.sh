for L in paper_1810_10197_b200/_lib/libsrk.so paper_1810_10197_b200/_lib_x1/libsrk.so; do
SRK_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:"k_project_tma|k_combine" --csv python tools/comb_timing.py 512 2>/dev/null | grep -E "k_project_tma|k_combine" | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
seen={}
for r in rows:
    k=r[4][:40]; m=r[-3]; v=r[-1]
    seen.setdefault((k,r[0]),{})[m]=v
import collections
agg=collections.OrderedDict()
for (k,i),d in seen.items():
    agg.setdefault(k,[]).append(d)
for k,l in agg.items():
    d=l[len(l)//2]
    print('$L'[-18:], k, {m:d[m] for m in d})
"
done
