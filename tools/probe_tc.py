import os, sys, torch, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
os.environ['LOUISKV_DEBUG'] = '1'
import paper_2510_11292_b200 as lkv
from synth.configs import C1, C2
from _pair import make_inputs
cfg = C1
inp = make_inputs(cfg, 1, 0, layout="blocked")
ctx = lkv.Context(lkv.make_config(cfg))
ctx.cluster_prompt(0, inp.K[0], inp.V[0])
print("C1", ctx.stats())
