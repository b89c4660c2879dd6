nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader > gpurun_out/${TAG}_bus.txt
python - >> gpurun_out/${TAG}_bus.txt <<'PY'
import torch
from cuda.bindings import runtime as rt
p = torch.cuda.get_device_properties(0)
print("sms", p.multi_processor_count)
PY
for kv in "FREEKV_X=0" "FREEKV_ATTN_EARLY=0" "FREEKV_ATTN_CLUSTER=4" "FREEKV_SELECT_NC=2" "FREEKV_SELECT_NC=1" "FREEKV_ATTN_CLUSTER=4;FREEKV_SELECT_NC=1"; do
  env $(echo $kv | tr ';' ' ') timeout 300 python bench.py --config c3 --steps 128 --no-extras --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/${TAG}_c3_${kv//[;=]/_}.json
done
