"""One BERT-Huge attention forward + backward (B = 1) for ncu captures."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.attn_bench import run  # noqa: E402

if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    run(f"bert-huge B={n}", n, 512, 20, 64, {})
