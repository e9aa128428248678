"""Build A/B variants of the library with extra -D flags (for timing experiments).

usage: python tools/ab.py TAG [DEFINE ...]   -> paper_2303_02346_b200/_ab/TAG/libflume_b200.so
run a variant with FLUME_B200_LIB=<that path> python bench.py ...
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2303_02346_b200.build import build_library  # noqa: E402

if __name__ == "__main__":
    print(build_library(defines=sys.argv[2:], tag=sys.argv[1]))
