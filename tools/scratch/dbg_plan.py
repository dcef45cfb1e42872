import sys, os
sys.path.insert(0, "/root/repo")


def main():
    os.environ["H2B_DEBUG_PLAN"] = "1"
    import __graft_entry__
    __graft_entry__.build()
    from paper_1811_05731_b200.workloads import build_workload
    from paper_1811_05731_b200.h2 import plan_view
    op, _ = build_workload(sys.argv[1], cache_dir="/tmp/h2b_cache", log=lambda m: None)
    for pf in (9216, 13312, 17408):
        P = plan_view(op, plan_flags=pf)
        print(pf, [(ph["mode"], ph["resident"], ph["res_max"], len(ph["unit0"]) - 1) for ph in P["phases"] if ph["mode"] == 1], flush=True)


if __name__ == "__main__":
    main()
