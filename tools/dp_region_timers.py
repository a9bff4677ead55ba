"""Write a copy of csrc/dp.cu with per-warp clock64() region timers (profiling
builds only; never committed as the product kernel).  Regions: prologue,
column setup, skip search, pair chunk (up to the candidate rounds), candidate
rounds + inserts, emit; summed over warps into counters[3..8], which the
PIPECUT_B200_DEBUG print shows as the 'frontier sizes' 0..5 entries.

    python tools/dp_region_timers.py src.cu out.cu
"""
import sys

s = open(sys.argv[1]).read()


def rep(old, new):
    global s
    assert old in s, old[:60]
    s = s.replace(old, new, 1)


rep("#define PC_DP_DIAG 0", "#define PC_DP_DIAG 0\n#define PCT() ((long long)clock64())")
rep("    uint32_t n_corner = 0, n_win = 0, n_rounds = 0, n_iters = 0;\n",
    "    uint32_t n_corner = 0, n_win = 0, n_rounds = 0, n_iters = 0;\n"
    "    long long t_pro = 0, t_col = 0, t_skip = 0, t_chk = 0, t_rnd = 0, t_emit = 0;\n"
    "    long long tz = PCT();\n")
rep("    if (s == 1) {\n        // level 0 holds", "    t_pro += PCT() - tz;\n    if (s == 1) {\n        // level 0 holds")
rep("rem = rem == 0 ? dpn - 1 : rem - 1) {\n", "rem = rem == 0 ? dpn - 1 : rem - 1) {\n            long long tc0 = PCT();\n")
rep("            int lim = bp_lo - 1;", "            t_col += PCT() - tc0;\n            int lim = bp_lo - 1;")
rep("            auto chunk = [&](int top, int ex_lo, int ex_hi) {\n",
    "            auto chunk = [&](int top, int ex_lo, int ex_hi) {\n                long long tk0 = PCT();\n")
rep("                const int cntw = whi - wlo + 1;\n",
    "                long long tk1 = PCT();\n                t_chk += tk1 - tk0;\n                const int cntw = whi - wlo + 1;\n")
rep("            };\n            const int ex_lo = 1, ex_hi = 0;",
    "                t_rnd += PCT() - tk1;\n            };\n            const int ex_lo = 1, ex_hi = 0;")
rep("                if (B.mono_skip && n > 0 && (int)n_ins != lim_v) {\n",
    "                if (B.mono_skip && n > 0 && (int)n_ins != lim_v) {\n                    long long ts0 = PCT();\n")
rep("                    lim_v = (int)n_ins;\n", "                    lim_v = (int)n_ins;\n                    t_skip += PCT() - ts0;\n")
rep("    // algorithmic work counters (one atomic per warp)\n",
    "    long long te0 = PCT();\n    // algorithmic work counters (one atomic per warp)\n")
rep("        if (ovf) atomicOr(B.overflow, 1);\n    }\n}\n",
    "        if (ovf) atomicOr(B.overflow, 1);\n    }\n    t_emit += PCT() - te0;\n"
    "    if (lane == 0) {\n"
    "        atomicAdd(&B.counters[3], (unsigned long long)t_pro);\n"
    "        atomicAdd(&B.counters[4], (unsigned long long)t_col);\n"
    "        atomicAdd(&B.counters[5], (unsigned long long)t_skip);\n"
    "        atomicAdd(&B.counters[6], (unsigned long long)t_chk);\n"
    "        atomicAdd(&B.counters[7], (unsigned long long)t_rnd);\n"
    "        atomicAdd(&B.counters[8], (unsigned long long)t_emit);\n    }\n}\n")
open(sys.argv[2], "w").write(s)
