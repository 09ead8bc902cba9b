for v in '{"mode":"f32"}' '{"mode":"f32","k_serpentine":1}' '{"mode":"f16"}' '{"mode":"f16","k_serpentine":1}' '{"mode":"f32","k_serpentine":1,"group_m":16}' '{"mode":"f32","k_serpentine":1,"group_m":4}'; do bash tools/ncu_metrics.sh "$v"; done
VARIANTS='[{"mode":"f32"},{"mode":"f32","k_serpentine":1},{"mode":"f16"},{"mode":"f16","k_serpentine":1}]' ROUNDS=6 python tools/ab.py
