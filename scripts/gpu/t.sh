python scripts/shard_step_time.py c3 c4 2>&1 | tail -12
