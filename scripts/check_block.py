import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_1802_08800_b200 as S
O = oracle.oracle()
ds = S.fixtures.sparse_classification(20000, 10000, 50.0, 20250810).rounded_f32()
for workers, gs, lanes in ((4096, 2048, 0), (4096, 2048, 32), (64, 32, 0), (8, 4, 0)):
    plan = S.parse_plan("row-ch:block:0"); plan.workers, plan.group_size, plan.lanes_per_worker = workers, gs, lanes
    hp = S.Hyperparams(alpha=0.1, batch_b=1, epochs=5, task=S.Task.SVM, step_decay=0.97)
    r = S.hogwild.train(S.Task.SVM, ds, hp, plan, 0)
    om, ol, _ = O.hogwild_serial(ds, 1, 0.1, 5, 0, 1, 0, workers, group_size=gs, decay=0.97)
    print(workers, gs, lanes, "gpu", [round(x, 1) for x in r.trace.losses()], "oracle", [round(x, 1) for x in ol],
          "rel", np.linalg.norm(r.model - om[-1]) / np.linalg.norm(om[-1]))
