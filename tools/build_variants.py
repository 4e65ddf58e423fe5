"""Build variants of libgicp_b200.so with extra -D flags for A/B timing (tools/ only).
usage: python tools/build_variants.py NAME:-DFOO=1,-DBAR=2 [NAME2:...]
-> paper_2308_07173_b200/variants/libgicp_NAME.so"""
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(HERE, "paper_2308_07173_b200"))
import build  # noqa: E402

os.makedirs(os.path.join(HERE, "paper_2308_07173_b200", "variants"), exist_ok=True)
for spec in sys.argv[1:]:
    name, _, flags = spec.partition(":")
    extra = [f for f in flags.split(",") if f]
    out = os.path.join(HERE, "paper_2308_07173_b200", "variants", f"libgicp_{name}.so")
    build.build(extra=extra, out=out)
    print("built", out)
