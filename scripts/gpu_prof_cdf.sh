mkdir -p gpurun_out
PF_PROFILE_FROM_STEP=200 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/steady_launches.csv python scripts/prof_run.py 24 210 > gpurun_out/steady.log 2>&1
python scripts/launch_summary.py gpurun_out/steady_launches.csv | head -25
PF_PROFILE_FROM_STEP=200 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"cdf_expand|cdf_reduce_qr" -c 4 -o gpurun_out/k4prof python scripts/prof_run.py 24 205 > gpurun_out/ncu_k4.log 2>&1
python scripts/ncu_summary.py gpurun_out/k4prof.ncu-rep | head -80
