"""Harness: run tools/tcgen05_peak (sustained tcgen05 tf32 / bf16 rate, >= 4 s each) while
sampling nvidia-smi clocks and throttle reasons; writes one JSON record (stdout)."""
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = []
q = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown"
smi = subprocess.Popen(["nvidia-smi", "--id=0", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "200"],
                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
th = threading.Thread(target=lambda: [rows.append(l.strip()) for l in smi.stdout], daemon=True)
th.start()
t0 = time.time()
out = subprocess.run([os.path.join(ROOT, "tools", "tcgen05_peak"), sys.argv[1] if len(sys.argv) > 1 else "4"],
                     capture_output=True, text=True).stdout
smi.terminate()
rec = json.loads(out.strip().splitlines()[-1])
sm = sorted(float(r.split(",")[0]) for r in rows if r and r.split(",")[0].strip().replace(".", "").isdigit())
rec.update({"raw_output": out.strip().splitlines()[:-1], "wall_s": round(time.time() - t0, 1),
            "clocks": {"sm_mhz_median": sm[len(sm) // 2] if sm else None, "sm_mhz_min": sm[0] if sm else None,
                       "samples": len(sm), "sw_power_cap_samples": sum(1 for r in rows if "Active" in r.split(",")[3]) if rows else 0},
            "method": "tools/tcgen05_peak.cu: 148 CTAs x 1 issuing thread, M128 N256 MMAs from SMEM (SW128 K-major), "
                      "2 alternating TMEM accumulators, loop calibrated to the requested seconds"})
print(json.dumps(rec, indent=1))
