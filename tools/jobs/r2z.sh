mkdir -p gpurun_out
(cd tools/ubench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atoms atoms.cu && ./atoms) > gpurun_out/r2z_atoms.txt 2>&1
