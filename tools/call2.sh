timeout 300 python tools/integ_time.py > gpurun_out/integ_time_base.txt 2>&1; tail -4 gpurun_out/integ_time_base.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_integrate_rows --launch-skip 10 --launch-count 1 -o gpurun_out/integ_p1_base python tools/integ_profile.py 12 codes > gpurun_out/ncu_integ.log 2>&1; tail -2 gpurun_out/ncu_integ.log
timeout 600 compute-sanitizer --tool initcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_initcheck.log 2>&1; grep "ERROR SUMMARY" gpurun_out/sanitize_initcheck.log
