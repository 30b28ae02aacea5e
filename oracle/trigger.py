"""Optimization Trigger — plain per-job decision rule.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

  1. drift first ("When the difference is larger than a certain threshold 10%. It will
     trigger the online adapting scheme"): |V_hat(cur) - V_bar| / V_bar > drift  -> ADAPT (2)
  2. gain ("skips that attempt if the gain is less than a certain threshold ... 5%"):
     best differs from cur and V_hat(best) - V_hat(cur) > gain * |V_hat(cur)|   -> RECONFIGURE (1)
  3. otherwise KEEP (0).
Gain is predicted-vs-predicted (both from the same inference pass); |cur| keeps the
rule meaningful for non-positive predictions (R#14).
"""
import math

KEEP, RECONFIGURE, ADAPT = 0, 1, 2


def trigger_decide(best_idx, best_score, cur_idx, cur_score, v_obs, gain=0.05, drift=0.10):
    out = []
    for j in range(len(best_idx)):
        b, s_b, c, s_c = int(best_idx[j]), float(best_score[j]), int(cur_idx[j]), float(cur_score[j])
        v = None if v_obs is None else float(v_obs[j])
        if v is not None and v > 0 and not math.isnan(s_c) and abs(s_c - v) / v > drift:
            out.append(ADAPT)
        elif b >= 0 and b != c and not math.isnan(s_b) and not math.isnan(s_c) and s_b - s_c > gain * abs(s_c):
            out.append(RECONFIGURE)
        else:
            out.append(KEEP)
    return out
