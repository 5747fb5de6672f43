#!/bin/bash
# projector: double-buffered cp.async taps (one barrier per class) -- parity
# tests with the new build, then same-box A/B of old vs new library builds
mkdir -p gpurun_out; L=gpurun_out/r2zc.log; : > $L
timeout 1500 python -m pytest tests/test_gpu_projector.py -q -p no:cacheprovider > gpurun_out/r2zc_pytest.log 2>&1
echo "projector pytest rc=$?" >> $L; tail -1 gpurun_out/r2zc_pytest.log >> $L
o=gpurun_out/r2zc.jsonl; : > $o
for rep in 1 2; do
  for lib in PROJOLD PROJNEW; do
    for psf in C2 C4; do
      LFBP_LIB_PATH=abtest/libhprime_$lib.so timeout 600 python tools/proj_bench.py --psf $psf --image 512 --iters 3 | sed "s/^{/{\"lib\": \"$lib\", /" >> $o 2>&1
    done
    LFBP_LIB_PATH=abtest/libhprime_$lib.so timeout 600 python tools/proj_bench.py --psf C1 --image 256 --iters 5 | sed "s/^{/{\"lib\": \"$lib\", /" >> $o 2>&1
  done
done
true
