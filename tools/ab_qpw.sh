# A/B of queries per warp (LCP_QPW) and warps per CTA (LCP_WPC_MIN) for the headline kernel; run via gpurun
for v in "1 1" "2 1" "4 1" "2 32" "1 1"; do set -- $v
  LCP_QPW=$1 LCP_WPC_MIN=$2 timeout 200 python bench.py --no-extras --cpu-budget-s 0.5 > gpurun_out/ab_q$1_w$2.log 2>&1
  python - "$1" "$2" <<'PY'
import json,sys
l=[x for x in open(f"gpurun_out/ab_q{sys.argv[1]}_w{sys.argv[2]}.log") if x.startswith("{")][-1]; d=json.loads(l)
print("QPW",sys.argv[1],"WPC",sys.argv[2],"value %.4g"%d["value"],"single_us %.3f"%(d["one_batch_in_flight"]["ms_per_step"]*1e3),"e2e %.4g"%d["e2e"]["value"], flush=True)
PY
done
