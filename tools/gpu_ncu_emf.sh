mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
PMHD_UPDATE=emf $CMD > gpurun_out/plain_emf.log 2>&1 && \
PMHD_UPDATE=emf ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:k_edge_emf|k_cell_update|k_update_fused" -c 12 --csv --log-file gpurun_out/emf_launches.csv $CMD > gpurun_out/ncu_emf.log 2>&1
python - <<'P'
import csv
rows=list(csv.reader([l for l in open("gpurun_out/emf_launches.csv") if not l.startswith("==")]))
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
for r in rows[1:]:
    if len(r)>vi: print(r[ii], r[ki][:40], r[mi], r[vi])
P
