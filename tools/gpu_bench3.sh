# three default bench runs back to back on one box (run-to-run and box-to-box spread)
O=gpurun_out/b3; mkdir -p $O; rm -f $O/*
nvidia-smi --query-gpu=name,pci.bus_id,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv > $O/smi.txt
for i in 1 2 3; do timeout 600 python bench.py 2>/dev/null | tail -1 > $O/bench$i.json; done
nvidia-smi --query-gpu=name,pci.bus_id,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv >> $O/smi.txt
