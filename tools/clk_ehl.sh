# Dev: sample SM clocks / power / throttle reasons with nvidia-smi while tools/time_ehl.py runs.
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 100 > gpurun_out/clk.log &
P=$!
python tools/time_ehl.py > gpurun_out/te.log 2>&1
kill $P
