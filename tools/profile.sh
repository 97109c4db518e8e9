#!/bin/bash
# Profiling pass run on the GPU box (one GPU):  gpurun -- 'bash tools/profile.sh <tag>'
# 1) launch list of one bench step (serialised, cold-cache per-launch times: compare SHARES)
# 2) ncu --set full captures of the top kernels (decode cluster GEMM, encoder GEMM, DLCL,
#    encoder attention, decoder attention).  Reports land in gpurun_out/.
tag=${1:-r1}
out=gpurun_out
mkdir -p $out
B="python bench.py --steps 1 --warmup 0 --chunk ${CHUNK:-3000} --no-e2e --no-cpu-baseline --no-paper-budget --no-c4 --workers 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-3000} --csv \
  --log-file $out/${tag}_launches.csv $B > $out/${tag}_launches.log 2>&1
echo "launches rc=$?"
full() {  # name regex, skip, count
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$2" -s $3 -c $4 \
    -o $out/${tag}_$1 -f $B > $out/${tag}_$1.log 2>&1
  echo "$1 rc=$?"
}
full dec_gemm '^k_gemm_tc$' 300 2
full enc_gemm '^k_gemm_tc$' 4 4
full dlcl '^k_dlcl_vec$' 10 1
full enc_attn '^k_attn_enc_tma$' 4 1
full dec_attn '^k_attn_(dec_self|cross)$' 20 2
