"""Phase-cycle breakdown of the enumeration (needs the -DBC_PHASE_PROF build:
python paper_2403_07858_b200/build.py --prof; run with BC_LIB=.../libbicount_b200_prof.so)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07858_b200 import synth, DeviceGraph, _abi
NAMES = ["claim", "level1-rebuild", "decode+map", "rows", "expand", "leaf-parents", "finish"]
name = sys.argv[1]
p, q = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else synth.CONFIGS[name][1][0]
from paper_2403_07858_b200 import EngineConfig
if name == "C5":
    dg = DeviceGraph.from_device_csr(*synth.fr_shaped_csr(device="cuda"))
    cfg = EngineConfig(batch_buffer_capacity=1 << 17)
else:
    dg = DeviceGraph(synth.build_config(name))
    cfg = EngineConfig()
L = _abi.load()
buf = (C.c_uint64 * 16)()
dg.count_raw(p, q, cfg)
L.bc_debug_phase_cycles(buf, 16)
rep, _ = dg.count_raw(p, q, cfg)
n = L.bc_debug_phase_cycles(buf, 16)
tot = sum(buf[i] for i in range(7))
print(f"{name} ({p},{q}) enum {rep.time_enum*1e3:.2f} ms; phase share of warp-cycles (n={n}):")
for i, nm in enumerate(NAMES):
    print(f"  {nm:15s} {100*buf[i]/max(tot,1):5.1f}%  {buf[i]/1e9:.3f} Gcyc")
