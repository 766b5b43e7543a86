# small problems: transpose vs a plain row copy of the same bytes (same launch mechanics: PDL, rotating buffers)
timeout 900 python scripts/exp_kernels.py --kernels tiled,copy,tma_tile --shapes 1024x1024:f64,2048x2048:f64,2048x4096:f64,3000x5000:f64,4096x4096:f64,8192x8192:f64,2048x2048:f32,4096x4096:f32,8192x8192:f32
