bash tools/cycle.sh r1o drt && bash tools/prof_nc.sh r1o drt 72 4
