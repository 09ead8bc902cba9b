VARIANTS='[{"mode":"f32"},{"mode":"f32","debug_flags":1},{"mode":"f32","debug_flags":2},{"mode":"f32","debug_flags":3}]' ROUNDS=4 python tools/ab.py
for v in '{"mode":"f32"}' '{"mode":"f32","debug_flags":1}' '{"mode":"f32","debug_flags":2}' '{"mode":"f32","debug_flags":3}'; do bash tools/ncu_metrics.sh "$v"; done
