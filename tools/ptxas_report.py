"""Compile every (dtype, NB) kernel translation unit with -Xptxas -v and report registers,
stack frame and spills per kernel (a stack frame means a register array was demoted to local
memory). Usage: python tools/ptxas_report.py [NB ...]"""
import concurrent.futures as cf
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2601_03754_b200", "csrc")
sizes = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 6, 8, 12, 16, 24, 32]


def one(args):
    dt, nb = args
    r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                        f"-DBTD_T={dt}", f"-DBTD_NB={nb}", "-c", os.path.join(CSRC, "btd_inst.cu"), "-o",
                        f"/tmp/ptxas_{dt}_{nb}.o", "-Xptxas", "-v"], capture_output=True, text=True)
    out = []
    for m in re.finditer(r"Compiling entry function '_ZN3btd\d+(\w+?)I\w+?Lb(\d)ELb(\d)E\S*?'.*?(\d+) bytes stack "
                         r"frame, (\d+) bytes spill stores, (\d+) bytes spill loads.*?Used (\d+) registers",
                         r.stderr, re.S):
        out.append(f"{dt:6s} NB={nb:2d} {m.group(1):22s} F{m.group(2)}S{m.group(3)} regs={m.group(7):3s} "
                   f"stack={m.group(4)} spill={m.group(5)}/{m.group(6)}")
    for m in re.finditer(r"Compiling entry function '_ZN3btd\d+(btd_level_bwd_kernel)\S*?'.*?(\d+) bytes stack "
                         r"frame, (\d+) bytes spill stores, (\d+) bytes spill loads.*?Used (\d+) registers",
                         r.stderr, re.S):
        out.append(f"{dt:6s} NB={nb:2d} {m.group(1):22s}      regs={m.group(5):3s} stack={m.group(2)} "
                   f"spill={m.group(3)}/{m.group(4)}")
    return "\n".join(out)


with cf.ThreadPoolExecutor(os.cpu_count()) as ex:
    for res in ex.map(one, [(dt, nb) for dt in ("float", "double") for nb in sizes]):
        print(res)
