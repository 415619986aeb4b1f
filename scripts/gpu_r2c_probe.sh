# r2c: sanity (GPU tests), a 10M config-3 line, then ncu --set full with source of the chain kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 600 python bench.py --config 3 --events 10000000 --steps 3 --warmup 3 --no-cpu --no-off > gpurun_out/r2c_cfg3_10M.json 2> gpurun_out/r2c_cfg3_10M.err; echo "bench rc=$?"
bash scripts/ncu_kernel_cfg3.sh r2c "k_window_run|k_window_verify|k_temporal_long|k_temporal_runs|k_readout|k_blur_prep|k_anchor2|k_link" 80 8
