"""Development: run the sharded parity case at 1 and 2 ranks (STG_SHARD_DEBUG
prints the reduced Gram checksums in call order)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

if __name__ == "__main__":
    import test_gpu_shard as t

    case = sys.argv[1] if len(sys.argv) > 1 else "rsvd_small"
    for w in (1, 2):
        try:
            t._run(w, case)
            print("PASS", w, flush=True)
        except AssertionError as e:
            print("FAIL", w, str(e)[:300], flush=True)
