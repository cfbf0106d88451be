"""Build a tuning variant of the engine into paper_1402_3788_b200/_lib/variants/ (selected at run
time with KM_LIB_VARIANT=<name>).  Usage: python tools/build_variant.py NAME DEFINE[=V] ..."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1402_3788_b200 import build

name, defines = sys.argv[1], sys.argv[2:]
out = build.LIBDIR / "variants" / f"libkmeans_b200_{name}.so"
out.parent.mkdir(parents=True, exist_ok=True)
print(build.build_engine(force=True, defines=defines, out=out))
