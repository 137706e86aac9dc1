"""C1 at 2^18 lanes: device time of the MAC-check class when the MAC check follows the online phase
immediately, after a host synchronize, and after a 2 ms host pause (profiles/r02s)."""
import sys, time
sys.path.insert(0, '.'); sys.argv = ['x']
exec(open('scripts/c1_small_probe.py').read().split('for lanes in')[0])
import torch
lanes = 1 << 18
inp = {"x": bc.rnd(lanes, 1), "y": bc.rnd(lanes, 2)}
for mode in ("plain", "sync_before_mac", "sleep_before_mac"):
    r = LocalRun(mul_graph(lanes), 2, profile_kernels=True)
    for k in range(4):
        r.deal(30 + k); r.bind_inputs(inp); r.share_inputs()
        r.online_begin()
        if mode == "sync_before_mac":
            torch.cuda.synchronize()
        elif mode == "sleep_before_mac":
            time.sleep(0.002)
        r.mac_check_launch()
        rep = r.mac_check()
        print(mode, round(rep.online_device_ms, 4), {n: round(v['ms'], 4) for n, v in rep.kstat.items() if v['launches']}, flush=True)
    r.close()
