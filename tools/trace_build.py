"""Rebuild libhexamoe.so with the debug timeline compiled in (or out with --off)."""
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_2411_01288_b200.build import CSRC, build  # noqa: E402

os.utime(os.path.join(CSRC, "umma.cu"))
build(extra=[] if "--off" in sys.argv else ["-DHXM_DBG_BUILD"] if "--dbg" in sys.argv else ["-DHXM_TRACE_BUILD"])
