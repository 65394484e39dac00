for a in "2**50 2**10" "2**50 2**20" "2**50 2**24" "2**48 2**32"; do
python tools/debug/one_call.py $a > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 0 --csv python tools/debug/one_call.py $a 2>/dev/null | grep -v "^==" > gpurun_out/g13_$(echo $a | tr ' *' '__').csv
done
ls gpurun_out/g13_*
