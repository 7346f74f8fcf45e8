"""Builds a product-flavour library variant with extra -D flags into ab_libs/ (for tools/ab.py A/B runs):
python tools/build_variant.py NAME -DFOO=1 ...  ->  ab_libs/libfdmoe_NAME.so"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_04667_b200 import build as b

name, flags = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(b.ROOT, "ab_libs"), exist_ok=True)
out = os.path.join(b.ROOT, "ab_libs", f"libfdmoe_{name}.so")
cmd = b._cmd(out, False, False)
cmd = cmd[:1] + flags + cmd[1:]
subprocess.run(cmd, check=True)
os.replace(out + ".tmp", out)
print(out)
