import sys, os
sys.path.insert(0, os.getcwd())
from paper_2511_18297_b200 import api
m = api.load_model("tests/golden/trained_csa8.asg1")
for w, c in [(64, 16), (256, 16), (512, 16), (1024, 2), (1024, 16)]:
    circ = api.gen_csa_multiplier(w)
    try:
        r = api.classify_aig(m, circ.aig, circ.labels, c)
        print(w, c, "ok", r.accuracy, flush=True)
    except Exception as e:
        print(w, c, "FAIL", e, flush=True)
        break
