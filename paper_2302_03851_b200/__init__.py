"""B200-native ED-Batch hot path (arXiv 2302.03851): C-ABI library libedbatch.so + ctypes binding.

    from paper_2302_03851_b200 import edbatch
    plan = edbatch.ed_plan(graphs, types, edbatch.fsm_from_priority(priority, len(types)))
    edbatch.ed_execute(plan, edbatch.DeviceWeights(types, params), edbatch.Workspace(plan))
"""
