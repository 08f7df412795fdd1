#!/bin/bash
# A/B bench session: parity tests, then short benches of variants.
mkdir -p gpurun_out
[ -z "$NO_PYTEST" ] && { timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; }
[ -z "$NO_PYTEST" ] && tail -4 gpurun_out/pytest_gpu.log
B="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e"
for v in "$@"; do
  case $v in
    split) PMHD_KERNELS=split $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    ldg) PMHD_UPDATE=ldg $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    m5ldg) PMHD_UPDATE=ldg $B --workload m5 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    b128ldg) PMHD_UPDATE=ldg $B --block 128 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    emf) PMHD_UPDATE=emf $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    emf-*) PMHD_UPDATE=emf PMHD_GPU_LIB=paper_1905_04341_b200/lib/exp/libpmhd_gpu_${v#emf-}.so $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    ex0) PMHD_EARLY_X1=0 $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    m5ex0) PMHD_EARLY_X1=0 $B --workload m5 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    conc*) PMHD_FLUX_CONC=${v#conc} $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    m5conc*) PMHD_FLUX_CONC=${v#m5conc} $B --workload m5 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    b128conc*) PMHD_FLUX_CONC=${v#b128conc} $B --block 128 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    default) $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    ovlpad*) PMHD_FACE_REUSE=0 PMHD_SLAB_PLANES=${v#ovlpad} PMHD_FLUX_SMEM_PAD=11776 $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    ovlnr*) PMHD_FACE_REUSE=0 PMHD_SLAB_PLANES=${v#ovlnr} $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    xy1) PMHD_FLUX_XY=2 $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    m5xy1) PMHD_FLUX_XY=2 $B --workload m5 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    xy) PMHD_FLUX_XY=1 $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    m5xy) PMHD_FLUX_XY=1 $B --workload m5 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    padonly) PMHD_FLUX_SMEM_PAD=11776 $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    sh_*) IFS=_ read -r _ a b c <<< "$v"; PMHD_ROW_SHIFT_ST=$a PMHD_ROW_SHIFT_FX=$b PMHD_ROW_SHIFT_EC=$c $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    shift*) PMHD_ROW_SHIFT=${v#shift} $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    slab*) PMHD_SLAB_PLANES=${v#slab} $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    notma) PMHD_TMA=0 $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    nooverlap) PMHD_OVERLAP=0 $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    ws) PMHD_UPDATE=ws $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    m5ws) PMHD_UPDATE=ws $B --workload m5 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    tma) PMHD_UPDATE=tma $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    m5tma) PMHD_UPDATE=tma $B --workload m5 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    nox1march) PMHD_FLUX_MARCH_X1=0 $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    both) PMHD_FLUX_MARCH_STAGES=3 $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    x1march) PMHD_FLUX_MARCH_X1=1 $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    m5x1march) PMHD_FLUX_MARCH_X1=1 $B --workload m5 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    st2) PMHD_FLUX_MARCH_STAGES=2 $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    st2x1) PMHD_FLUX_MARCH_STAGES=2 PMHD_FLUX_MARCH_X1=1 $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    m5st2x1) PMHD_FLUX_MARCH_STAGES=2 PMHD_FLUX_MARCH_X1=1 $B --workload m5 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    tile) PMHD_FLUX_MARCH=0 $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    m5tile) PMHD_FLUX_MARCH=0 $B --workload m5 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    noreuse) PMHD_FACE_REUSE=0 $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    m5) $B --workload m5 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    m5noreuse) PMHD_FACE_REUSE=0 $B --workload m5 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    b128) $B --block 128 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    b128noreuse) PMHD_FACE_REUSE=0 $B --block 128 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    hlle|roe) $B --riemann $v > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    *-hlle|*-roe) PMHD_GPU_LIB=paper_1905_04341_b200/lib/exp/libpmhd_gpu_${v%-*}.so $B --riemann ${v##*-} > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    parity) PMHD_GPU_LIB=paper_1905_04341_b200/lib/libpmhd_gpu_parity.so $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    m*) PMHD_GPU_LIB=paper_1905_04341_b200/lib/exp/libpmhd_gpu_$v.so $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    r_*) PMHD_GPU_LIB=paper_1905_04341_b200/lib/exp/$v/libpmhd_gpu.so $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
    *) PMHD_GPU_LIB=paper_1905_04341_b200/lib/exp/libpmhd_gpu_$v.so $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err ;;
  esac
  python - "$v" <<'PY'
import json,sys
v=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/ab_{v}.json"))
    r=d["roofline"]
    print(f"{v:10s} cups={d['value']:.4g} ms/step={d['ms_per_step']:.3f} flux_ms={r['kernel'].split('avg ')[1].split(' ms')[0]} upd_ms={r['update_kernel']['avg_ms']:.3f} flux_fp64={r['frac']:.3f} cyc_fp64={r['fp64_whole_cycle']['frac']:.3f} shares={ {k:round(x,3) for k,x in r['region_share'].items()} } clk={d['clocks']}")
except Exception as e:
    print(v, "FAILED", e, open(f"gpurun_out/ab_{v}.err").read()[-500:])
PY
done
