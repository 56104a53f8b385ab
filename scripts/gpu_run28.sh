set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hbm_read scripts/micro/hbm_read.cu && timeout 120 /tmp/hbm_read
