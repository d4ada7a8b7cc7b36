# Profiles of the bench step (run under gpurun): launch list of 2 timed steps, and one
# --set full capture of the tcgen05 fwd/dgrad launches (incl. the fused conv+pool) of one step.
# The launch list covers the 3 warm-up + 2 timed steps: summarise with `python tools/ncu_summary.py launches.csv 5`.
python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu-baseline --sustain-s 0 > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu-baseline --sustain-s 0 > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"tc_fwd_tr|tc_fwd_vpair|tc_conv_fwd|tc_conv_maxpool" \
    -s 30 -c 10 -o gpurun_out/tcfwd_step python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline --sustain-s 0 \
    > gpurun_out/ncu_full.log 2>&1
