import cProfile, pstats, io, sys, os
sys.path.insert(0, os.getcwd())
import benchlib.configs as C
pr = cProfile.Profile()
pr.enable()
r = C.c1_routed(reference=False, reps=3)
pr.disable()
print(r["value"], r["runs"])
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue()[:6000])
