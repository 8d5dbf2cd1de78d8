import json, sys
sys.path.insert(0, ".")
from benchlib import configs as C
r = C.c3_kv(6539.2)
print(json.dumps(r))
