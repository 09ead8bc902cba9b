VARIANTS='[{"mode":"f32"},{"mode":"f32","l2_hints":-1},{"mode":"f16"},{"mode":"f16","l2_hints":-1}]' python tools/ab.py
for v in '{"mode":"f32"}' '{"mode":"f32","l2_hints":-1}' '{"mode":"f16"}' '{"mode":"f16","l2_hints":-1}'; do bash tools/ncu_metrics.sh "$v"; done
