mkdir -p gpurun_out
for B in 1 32; do
timeout 300 ncu --set full --clock-control none -s 20 -c 1 -o gpurun_out/cublas_b$B python tools/exp_cublas.py $B > /dev/null 2>&1
ncu -i gpurun_out/cublas_b$B.ncu-rep --page details --csv > gpurun_out/cublas_b$B.details.csv 2>/dev/null
ncu -i gpurun_out/cublas_b$B.ncu-rep --page raw --csv > gpurun_out/cublas_b$B.raw.csv 2>/dev/null
rm -f gpurun_out/cublas_b$B.ncu-rep
done
