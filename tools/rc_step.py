"""Racecheck helper: two fused steps on an n-element flat buffer (usage: rc_step.py n kind)."""
import sys, torch
sys.path.insert(0, '.')
import paper_2110_02861_b200 as q8, synth
n = int(sys.argv[1]); kind = sys.argv[2]
p = synth.params(n).cuda(); g = synth.grads(n, step=1, dtype="bfloat16").cuda()
s1, a1 = synth.zero_state(n, device="cuda"); s2, a2 = synth.zero_state(n, device="cuda")
for t in (1, 2):
    q8.optim8bit_step(kind, p, g, s1, s2, a1, a2, step=t, **synth.HPARAMS[kind])
torch.cuda.synchronize(); print("ok", n, kind)
