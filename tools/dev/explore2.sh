set -x
python tools/synth_explore.py --n 32768 --cfg '{"sink_strength": 41, "anchor_strength": 36}' --taus '[[0.3,0.5],[0.5,0.7],[0.7,0.85],[0.8,0.9],[0.9,0.95]]'
python tools/synth_explore.py --n 32768 --cfg '{"sink_strength": 41, "anchor_strength": 36, "n_stripes": 1, "stripe_planes": 16, "stripe_amp": 3.3}' --taus '[[0.3,0.5],[0.5,0.7],[0.7,0.85],[0.8,0.9],[0.9,0.95]]'
python tools/synth_explore.py --n 32768 --cfg '{"sink_strength": 41, "anchor_strength": 36, "noise_sigma": 0.8}' --taus '[[0.3,0.5],[0.5,0.7],[0.7,0.85],[0.8,0.9],[0.9,0.95]]'
python tools/synth_explore.py --n 131072 --cfg '{"sink_strength": 41, "anchor_strength": 36}' --taus '[[0.3,0.5],[0.5,0.7],[0.7,0.85],[0.8,0.9],[0.9,0.95]]'
