timeout 60 ./build/dbg_bulk t 128 0 > gpurun_out/dbg3.log 2>&1; echo rc=$?
grep -v "kt" gpurun_out/dbg3.log | tail; grep "kt" gpurun_out/dbg3.log | tail -40
