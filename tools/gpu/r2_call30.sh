nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/param_launch tools/micro/param_launch.cu && /tmp/param_launch
