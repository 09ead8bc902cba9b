VARIANTS='[{"mode":"f32"},{"mode":"f32","promote_k":-1},{"mode":"f16"}]' ROUNDS=4 python tools/ab.py
for v in '{"mode":"f32"}' '{"mode":"f32","promote_k":-1}' '{"mode":"f16"}'; do bash tools/ncu_metrics.sh "$v"; done
