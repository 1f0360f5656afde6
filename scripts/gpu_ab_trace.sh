# per-variant PASE_TRACE timelines of one workload: gpurun_out/trace_<wl>_<k>.npy (k = variant index)
cd $GRAFT_REPO_ROOT
W=${W:-transformer_le}
IFS=';' read -ra VS <<< "${VARIANTS:-base;PASE_NO_2D=1}"
k=0
for v in "${VS[@]}"; do
  envs=""; [ "$v" != "base" ] && envs="$v"
  env $envs timeout 600 python scripts/trace_run.py $W > gpurun_out/trace_${W}_$k.log 2>&1
  mv gpurun_out/trace_$W.npy gpurun_out/trace_${W}_$k.npy
  echo "[$k] $v: $(grep 'dp phase' gpurun_out/trace_${W}_$k.log)"
  k=$((k+1))
done
