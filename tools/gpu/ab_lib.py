"""A/B helper: run tools/profile_step.py against another build of the library (argv[1])."""
import runpy
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2412_15840_b200 as nds
nds.load_library(os.path.abspath(sys.argv[1]))
sys.argv = ["profile_step.py"] + sys.argv[2:]
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profile_step.py"), run_name="__main__")
