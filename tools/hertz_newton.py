import sys; sys.path.insert(0,'/root/repo')
from paper_2605_24339_b200 import scenes as S, system as SY
s,_=SY.build_hertz_system(S.HertzConfig(refine=0.7))
ms,pcg=s.time_newton(SY.SolverSettings(),3)
print(ms,pcg)
