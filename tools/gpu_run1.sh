set -x
nproc; free -g | head -2
python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; tail -15 gpurun_out/gputest.log
python bench.py > gpurun_out/bench_R.json 2> gpurun_out/bench_R.err; tail -3 gpurun_out/bench_R.err
python bench.py --config C5 --steps 5 --warmup 2 --no-cpu > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; tail -3 gpurun_out/bench_C5.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -3 gpurun_out/bench_ref.err
