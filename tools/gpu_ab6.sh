for v in '{"mode":"f32"}' '{"mode":"f32","config":6}' '{"mode":"f32","config":6,"promote_k":-1}' '{"mode":"f16","config":6}'; do bash tools/ncu_metrics.sh "$v"; done
