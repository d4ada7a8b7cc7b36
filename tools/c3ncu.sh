# ncu captures of the config-3 fp32 kernels (development)
for op in "$@"; do
  python tools/one_op_c3.py $op 2 > gpurun_out/plain_$op.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"f32_wgrad_kernel|tiled|c1_fwd|plane|n1s2" -s 1 -c 1 -o gpurun_out/c3_$op python tools/one_op_c3.py $op 2 > gpurun_out/ncu_$op.log 2>&1
done
