set -x
O=gpurun_out/s4; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "tests rc=$?" >> $O/gputest.log
timeout 600 python bench.py > $O/bench5.json 2> $O/bench5.err
