"""A/B of the configs[2] batched adaptive sweep (bench.config2; development aid, VTRAIN_B200_LIB picks the build)."""
import json, os, sys
sys.path.insert(0, ".")
import bench
r = bench.config2()
print(os.environ.get("TAG", ""), json.dumps({k: r[k] for k in ("ms_per_sweep", "ms_per_sweep_eager")}))
