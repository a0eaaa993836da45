python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/gputest12.log
python tools/run_rpca.py > gpurun_out/rpca_plain.log 2>&1
python tools/run_corutv.py c2 5 > gpurun_out/c2_plain.log 2>&1
python tools/run_corutv.py c1 5 > gpurun_out/c1_plain.log 2>&1
for l in 50 110; do
  python tools/small_sweep.py $l > gpurun_out/sw_$l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sw_$l.csv python tools/small_sweep.py $l > /dev/null 2>&1
done
python tools/run_rpca.py > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 5200 -c 4000 --csv --log-file gpurun_out/launches_rpca_alm.csv python tools/run_rpca.py > /dev/null 2>&1
