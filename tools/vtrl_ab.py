"""A/B of the packed .vtrl codec pair at 2^26 (bench.vtrl_codec; development aid, VTRAIN_B200_LIB picks the build)."""
import json, os, sys
sys.path.insert(0, ".")
import bench
r = bench.vtrl_codec(int(sys.argv[1]) if len(sys.argv) > 1 else 26)
print(os.environ.get("TAG", ""), json.dumps({k: r[k] for k in ("round_log_packed_frac", "replay_packed_frac", "auditor_equals_trainer_bitwise")}))
