"""Run N eager steps of a benchmark program (for ncu launch lists / captures)."""
import argparse
import sys

sys.path.insert(0, ".")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--program", default="c2_tf8_dense")
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    from paper_2401_11202_b200.programs import load_program, synthetic_inputs
    from paper_2401_11202_b200.session import Session
    p = load_program(args.program)
    sess = Session(p.dense if p.local is None else p.local, p.sharding)
    sess.load(synthetic_inputs(p.dense, seed=0, scale=0.02))
    for _ in range(args.steps):
        sess.run()
    sess.sync()
    print("records", sess.ex.plan.n_records, "launches/step", sess.launch_count())


if __name__ == "__main__":
    main()
