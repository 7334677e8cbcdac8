for t in 1 2 3 4 6; do echo "target=$t $(EKV_ATTN_TARGET=$t python tools/time_prefill.py 2>&1 | grep 'U=16')"; done
