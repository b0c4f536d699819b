"""Build a copy of the package with extra nvcc defines into <dir> (for same-box A/B runs):
    python tools/dev/build_variant.py _exp_x -DVSP_POLY_MASK=0u"""
import os, shutil, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
dst_root = os.path.join(ROOT, sys.argv[1])
shutil.rmtree(dst_root, ignore_errors=True)
shutil.copytree(os.path.join(ROOT, "paper_2603_04460_b200"), os.path.join(dst_root, "paper_2603_04460_b200"),
                ignore=shutil.ignore_patterns("_objs", "*.so", "__pycache__"))
shutil.copytree(os.path.join(ROOT, "include"), os.path.join(dst_root, "include"))
sys.path.insert(0, dst_root)
from paper_2603_04460_b200 import _build  # the copy
_build.FLAGS.extend(sys.argv[2:])
print(_build.build())
