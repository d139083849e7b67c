"""Run the seeded fuzz configurations for many seeds (one-off stress run):
    python tools/fuzz_many.py START COUNT"""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_fuzz as f  # noqa: E402

start, count = int(sys.argv[1]), int(sys.argv[2])
bad = 0
for seed in range(start, start + count):
    for fn in (f.test_random_configuration_matches_oracle, f.test_random_engine_step_matches_oracle):
        try:
            fn(seed)
        except Exception:  # noqa: BLE001
            bad += 1
            print(f"FAIL {fn.__name__} seed {seed}")
            traceback.print_exc(limit=2)
print(f"done: {2 * count} cases, {bad} failures")
