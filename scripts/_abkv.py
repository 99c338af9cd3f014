import ctypes, os, sys, runpy
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_03474_b200 import _native as N
lib = ctypes.CDLL(str(N.LIB_PATH)); N.ABI_VERSION = lib.rld_abi_version()
sys.argv = ["kv_profile.py"] + sys.argv[1:]
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "kv_profile.py"), run_name="__main__")
