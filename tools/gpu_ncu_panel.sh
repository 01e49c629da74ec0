mkdir -p gpurun_out
./build/panel_bench > gpurun_out/pb_plain.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pb_kernel -s 0 -c 1 -o gpurun_out/prof_panel ./build/panel_bench > gpurun_out/ncu_panel.log 2>&1; echo "ncu rc=$?"; cat gpurun_out/pb_plain.log
