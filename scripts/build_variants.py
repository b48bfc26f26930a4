"""Build A/B variants of the extension: build/variants/NAME.so with extra -D switches.
usage: python scripts/build_variants.py NAME=DEF1,DEF2 ...   (DEF like CHAM_LOOK=0)"""
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2411_17741_b200.csrc.build import build  # noqa: E402


def one(spec):
    name, defs = spec.split("=", 1)
    out = ROOT / "build" / "variants" / f"{name}.so"
    out.parent.mkdir(parents=True, exist_ok=True)
    return build(force=True, out=out, defines=tuple(defs.split(",")))


if __name__ == "__main__":
    with ThreadPoolExecutor(4) as ex:
        for p in ex.map(one, sys.argv[1:]):
            print(p)
