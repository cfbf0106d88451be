# per-step device/host trace of km_lloyd calls (cfg3) + ncu launch list of one T=20 call
mkdir -p gpurun_out
KM_CALL_TRACE=1 timeout 300 python tools/time_call.py cfg3 > gpurun_out/r4c_call.txt 2> gpurun_out/r4c_trace.txt
cat gpurun_out/r4c_call.txt
awk 'NR%20==10' gpurun_out/r4c_trace.txt | head -8
cat > /tmp/one.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np
from paper_1402_3788_b200 import _native
from paper_1402_3788_b200.datasets import generate_synthetic_array
x = generate_synthetic_array(2_000_000, 25, 16, seed=0, dtype=np.float32)
e = _native.NativeEngine(0); e.load(x)
for T in (20, 20, 1):
    e.lloyd(x[:16].astype(np.float64), T, 0.0, want_labels=False)
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4c_launches.csv python /tmp/one.py > /dev/null 2>&1
grep -v "^==" gpurun_out/r4c_launches.csv | awk -F'","' '{print $5, $NF}' | tail -20
