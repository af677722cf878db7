# ncu captures of the two slowest one-CTA kernels of a config-2 step: the TSQR
# leaf of the exact residual norm and the 12-column rounding SVD.
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"wqr_kernel<\(int\)12, \(int\)2|svd_warp_kernel<\(int\)8, \(int\)12|wqr_kernel<\(int\)4, \(int\)2" --launch-skip 6 -c 6 \
  -o gpurun_out/r02i_qr_svd python tools/march_hash.py 2 --steps 5 > gpurun_out/r02i_ncu_qr.log 2>&1
tail -3 gpurun_out/r02i_ncu_qr.log
ls -la gpurun_out/r02i_qr_svd.ncu-rep
