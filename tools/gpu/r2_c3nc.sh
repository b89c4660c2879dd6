nvidia-smi --query-gpu=name,serial,pci.bus_id --format=csv > gpurun_out/${TAG}_gpu.txt
for i in 1 2; do for nc in 8 4 2; do
  FREEKV_SELECT_NC=$nc timeout 300 python bench.py --config c3 --steps 128 --no-extras --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/${TAG}_c3_nc${nc}_$i.json
done; done
