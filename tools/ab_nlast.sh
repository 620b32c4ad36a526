export SPARTON_DEV=1   # the library honours SPARTON_* switches only under this gate
python -m pytest tests/test_gpu_forward.py tests/test_gpu_backward.py -x -q 2>&1 | tail -2
mkdir -p gpurun_out
for S in 100 300 384 512; do
  for lib in build/ab/base.so build/ab/nlast.so; do SPARTON_LIB=$lib python tools/fwd_time.py 128 $S 768 250002 "S=$S $lib"; done
done
