import sys, numpy as np
sys.path.insert(0,'.')
from paper_2501_19013_b200.setup.geometry import BallVoids
from paper_2501_19013_b200.setup.grid import Grid
from paper_2501_19013_b200.setup.problem import ScmProblem
p=int(sys.argv[1]); n_e=int(sys.argv[2])
geom = BallVoids(2, [[0.5, 0.5], [0.15, 0.8]], [0.27, 0.1])
prob = ScmProblem.build(Grid.build(geom, "lagrange", p, n_e), 1e-3, 2)
K = prob.csr_stiffness(); op = prob.device_operator()
x = np.random.default_rng(p).standard_normal(prob.n_dof)
y=op@x; print(p, n_e, np.linalg.norm(y-K@x)/np.linalg.norm(K@x))
