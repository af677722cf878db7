# ncu passes of round 2, final kernels (run each only after the plain command exited 0):
#  1. launch list of config-2 steps 11-12 (gpu__time_duration per launch)
#  2. full capture of the Gauss-Jordan kernel at N = 792, 1155, 1848
set -x
python tools/time_march.py 2 12 > gpurun_out/r02i_time_march.log 2>&1 || exit 1
T2S2_PROFILE_FROM=11 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02i_launches_steps11_12.csv python tools/time_march.py 2 12 > gpurun_out/r02i_ncu_launch.log 2>&1
python tools/gj_profile.py 792 1155 1848 > gpurun_out/r02i_gj_profile.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:gj_kernel -c 3 -o gpurun_out/r02i_gj_sizes \
  python tools/gj_profile.py 792 1155 1848 > gpurun_out/r02i_ncu_gj.log 2>&1
ls -la gpurun_out/r02i_*
