import json, random, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from oracle import ref
from paper_2602_11686_b200 import planner as PP
from test_oracle_exact import _cfg, _instances
rng = random.Random(int(sys.argv[1]))
ok = mism = err = 0
for n, e, c, nodes, R in _instances(3000, rng):
    kw = {}
    if rng.random() < 0.1: kw["max_layouts"] = rng.randint(1, 10)
    if rng.random() < 0.1: kw["gran"] = 1
    cfg = _cfg(n, e, c, nodes=nodes, seed=rng.randint(0, 99), eps=rng.choice([2, 3, 4]), f_ckpt=rng.choice([0, 1]), **kw)
    inst = json.dumps({"R": R})
    try:
        theirs = ref.oracle_gap_json(ref.config(cfg), inst)
    except ref.RefError:
        err += 1
        continue
    mine = PP.oracle_gap_json(PP.Config(cfg), inst)
    if mine == theirs: ok += 1
    else:
        mism += 1
        if mism < 4: print("MISMATCH", cfg, inst, mine, theirs)
print("ok", ok, "mismatch", mism, "ref errors", err)
# simulate with oracle_layout, several traces
sm = 0
for s in range(40):
    spec = json.dumps({"n_devices": rng.choice([2, 4]), "n_experts": 4, "n_layers": 2, "n_iterations": 4, "tokens_per_device": rng.choice([8, 12, 16]),
                       "skew_alpha": rng.choice([0.3, 1.0]), "drift_sigma": 0.3, "seed": s})
    n = json.loads(spec)["n_devices"]
    cfg = _cfg(n, 4, 2, seed=s)
    try:
        theirs = ref.simulate(ref.config(cfg), ref.trace_generate(spec), "laer,oracle_layout")
    except ref.RefError:
        continue
    mine = PP.simulate(PP.Config(cfg), PP.Trace.generate(spec), "laer,oracle_layout")
    sm += mine != theirs
print("simulate mismatches", sm)
