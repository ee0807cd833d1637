PYTHONPATH=. ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_exact -s 10 -c 5 --csv --log-file gpurun_out/exb_new.csv python bench.py --steps 1 --warmup 2 --no-cpu > /dev/null 2>&1
python tools/latency.py 2>&1 | head -2
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
