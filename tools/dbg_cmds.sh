for c in "32 3 1 1 fwd" "32 3 1 1 inv" "32 3 32 1 fwd" "32 3 32 1 inv" "32 3 1 0 fwd" "32 3 1 0 inv" "32 8 1 1 fwd" "32 8 1 1 inv" "32 10 1 1 fwd" "32 10 1 1 inv" "64 3 1 1 fwd" "64 3 1 1 inv"; do
  CUDA_LAUNCH_BLOCKING=1 timeout 60 python tools/dbg_small.py $c 2>&1 | tail -1
done
