import cProfile, pstats, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1810_05762_b200.policy import ActorCritic
from paper_1810_05762_b200.ppo import PPOConfig, PPOLearner
torch.manual_seed(0)
B, O, A = 32768, 76, 21
m = ActorCritic(O, A).cuda()
L = PPOLearner(m, PPOConfig(frames_per_iter=8))
xw = torch.randn(B, O, device="cuda"); act = torch.randn(B, A, device="cuda")
adv = torch.randn(B, device="cuda"); ret = torch.randn(B, device="cuda")
st = torch.stack([torch.tensor(float(B), dtype=torch.float64), adv.double().sum().cpu(), (adv.double()**2).sum().cpu()]).cuda()
for _ in range(3): L.update(xw, act, None, adv, ret, adv_stats=st)
torch.cuda.synchronize()
pr = cProfile.Profile(); t0 = time.perf_counter(); pr.enable()
for _ in range(5): L.update(xw, act, None, adv, ret, adv_stats=st)
torch.cuda.synchronize(); pr.disable()
print("per update", (time.perf_counter() - t0) / 5)
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
