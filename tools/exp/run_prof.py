# phase timing of k_pipe2 configurations at 2^16 (tools/exp/exp_prof.cu): per task (group 0, thread 0) cycles
# waiting for the staged tile and computing it, by task kind; release warp: waiting for done, fence + red
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["EXP_LIB"] = "libprof.so"
sys.argv = [sys.argv[0], sys.argv[1] if len(sys.argv) > 1 else "0,1"]
exec(open(os.path.join(ROOT, "tools", "exp", "run_wide.py")).read().replace("for i in cfgs:", "for i in cfgs:\n    lib.exp_prof_zero()"), globals())
