"""Run bench.py against another build of the engine (A/B on the same box):
    python tools/bench_with_lib.py path/to/libcpfast_b200.so [bench args...]"""
import runpy
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1205_2584_b200 import _native

_native.LIB_PATH = Path(sys.argv[1]).resolve()
sys.argv = ["bench.py"] + sys.argv[2:]
runpy.run_path(str(Path(__file__).resolve().parents[1] / "bench.py"), run_name="__main__")
